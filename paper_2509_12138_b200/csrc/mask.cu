// K11 background-mask renderer (sm_100a): render_mask (render.hpp:210-233).
//
// One thread per cloud point: exact fp64 projection (no FMA contraction, the
// reference's x86-64 evaluation order), then the disc of radius
// footprint+dilation is stamped into a byte mask. Stores are idempotent
// (every writer writes 1), so overlapping discs need no atomics and the mask
// is bit-exact.
#include "dsg_internal.h"
#include "raster.h"

namespace dsg {

namespace {

__global__ void __launch_bounds__(256) k_render_mask(const double* __restrict__ pts, int64_t n,
                                                     CamDev c, double radius, double radius_sq,
                                                     uint8_t* __restrict__ mask) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d0 = ds(pts[3 * i], c.pos[0]), d1 = ds(pts[3 * i + 1], c.pos[1]);
  double d2 = ds(pts[3 * i + 2], c.pos[2]);
  double tx = da(da(dm(c.R[0], d0), dm(c.R[1], d1)), dm(c.R[2], d2));
  double ty = da(da(dm(c.R[3], d0), dm(c.R[4], d1)), dm(c.R[5], d2));
  double tz = da(da(dm(c.R[6], d0), dm(c.R[7], d1)), dm(c.R[8], d2));
  if (tz <= c.near_plane) return;
  double u = da(c.half_w, dd(dm(c.f, tx), tz));
  double v = ds(c.half_h, dd(dm(c.f, ty), tz));
  int x0 = max(0, to_int_x86(ceil(ds(ds(u, radius), 0.5))));
  int x1 = min(c.width - 1, to_int_x86(floor(ds(da(u, radius), 0.5))));
  int y0 = max(0, to_int_x86(ceil(ds(ds(v, radius), 0.5))));
  int y1 = min(c.height - 1, to_int_x86(floor(ds(da(v, radius), 0.5))));
  for (int y = y0; y <= y1; ++y)
    for (int x = x0; x <= x1; ++x) {
      double dx = ds(da((double)x, 0.5), u);
      double dy = ds(da((double)y, 0.5), v);
      if (da(dm(dx, dx), dm(dy, dy)) <= radius_sq) mask[(int64_t)y * c.width + x] = 1;
    }
}

}  // namespace

void render_mask_dev(const double* pts, int64_t n, const CamDev& cam, double radius,
                     uint8_t* mask, cudaStream_t st) {
  if (n <= 0) return;
  k_render_mask<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pts, n, cam, radius, radius * radius,
                                                              mask);
                                                              count_launch();
  DSG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace dsg
