// Grid-hash k-nearest-neighbour seeding (sm_100a): knn_mean_distances,
// median_nn_spacing, seed_gaussians(Knn) and ground_truth_model (seed.hpp).
//
// The reference is brute force O(N^2) (seed.hpp:16-35), ~50 s at 100K and
// infeasible at 4M+. Here points are bucketed into a uniform grid (cell edge
// h), sorted by cell key with the onesweep sort, and each point scans
// Chebyshev rings of cells around its own until its k-th best distance is
// <= r*h (every unvisited point is farther than that), which makes the
// result exact. Distances are the reference's fp64 (p_i - p_j).norm()
// without FMA contraction, and the k smallest are summed in ascending order
// (seed.hpp:29-32), so means are bit-identical to the reference.
#include <algorithm>
#include <cmath>
#include <vector>

#include "dsg_internal.h"
#include "raster.h"

namespace dsg {

namespace {

constexpr int kMaxK = 16;

struct Grid {
  double lo[3];
  double h;
  int64_t dims[3];
};

__device__ __forceinline__ uint64_t cell_key(int64_t cx, int64_t cy, int64_t cz, const Grid& g) {
  return (uint64_t)((cz * g.dims[1] + cy) * g.dims[0] + cx);
}

__device__ __forceinline__ int64_t cell_coord(double v, double lo, double h, int64_t dim) {
  int64_t c = (int64_t)floor((v - lo) / h);
  return c < 0 ? 0 : (c >= dim ? dim - 1 : c);
}

__global__ void k_cell_keys(const double* __restrict__ p, int64_t n, Grid g, uint64_t* keys,
                            uint32_t* idx) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t cx = cell_coord(p[3 * i], g.lo[0], g.h, g.dims[0]);
  int64_t cy = cell_coord(p[3 * i + 1], g.lo[1], g.h, g.dims[1]);
  int64_t cz = cell_coord(p[3 * i + 2], g.lo[2], g.h, g.dims[2]);
  keys[i] = cell_key(cx, cy, cz, g);
  idx[i] = (uint32_t)i;
}

// First position of `key` in the sorted key array (or -1).
__device__ __forceinline__ int64_t find_cell(const uint64_t* __restrict__ keys, int64_t n,
                                             uint64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && keys[lo] == key) ? lo : -1;
}

__global__ void __launch_bounds__(128) k_knn(const double* __restrict__ p, int64_t n, Grid g,
                                             const uint64_t* __restrict__ skeys,
                                             const uint32_t* __restrict__ sidx, int k,
                                             double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double px = p[3 * i], py = p[3 * i + 1], pz = p[3 * i + 2];
  const int64_t cx = cell_coord(px, g.lo[0], g.h, g.dims[0]);
  const int64_t cy = cell_coord(py, g.lo[1], g.h, g.dims[1]);
  const int64_t cz = cell_coord(pz, g.lo[2], g.h, g.dims[2]);
  double best[kMaxK];
  for (int m = 0; m < k; ++m) best[m] = INFINITY;
  const int kk = (int)(n - 1 < (int64_t)k ? n - 1 : (int64_t)k);
  if (kk <= 0) {
    out[i] = 0.0;
    return;
  }
  const int64_t maxr = max(g.dims[0], max(g.dims[1], g.dims[2]));
  for (int64_t r = 0; r <= maxr; ++r) {
    for (int64_t dz = -r; dz <= r; ++dz) {
      int64_t z = cz + dz;
      if (z < 0 || z >= g.dims[2]) continue;
      for (int64_t dy = -r; dy <= r; ++dy) {
        int64_t y = cy + dy;
        if (y < 0 || y >= g.dims[1]) continue;
        bool shell_yz = (dz == -r || dz == r || dy == -r || dy == r);
        int64_t step = shell_yz ? 1 : 2 * r;  // interior rows: only the two x end cells
        for (int64_t dx = -r; dx <= r; dx += (step == 0 ? 1 : step)) {
          int64_t x = cx + dx;
          if (x < 0 || x >= g.dims[0]) continue;
          int64_t s = find_cell(skeys, n, cell_key(x, y, z, g));
          if (s < 0) continue;
          const uint64_t key = skeys[s];
          for (; s < n && skeys[s] == key; ++s) {
            uint32_t j = sidx[s];
            if (j == (uint32_t)i) continue;
            double ex = ds(px, p[3 * j]), ey = ds(py, p[3 * j + 1]), ez = ds(pz, p[3 * j + 2]);
            double d = sqrt(da(da(dm(ex, ex), dm(ey, ey)), dm(ez, ez)));
            if (d < best[kk - 1]) {
              int m = kk - 1;
              while (m > 0 && best[m - 1] > d) {
                best[m] = best[m - 1];
                --m;
              }
              best[m] = d;
            }
          }
        }
      }
    }
    // all unvisited points are at least r*h away
    if (best[kk - 1] < (double)r * g.h * (1.0 - 1e-12)) break;
  }
  double s = 0.0;
  for (int m = 0; m < kk; ++m) s = da(s, best[m]);
  out[i] = dd(s, (double)kk);
}

__global__ void k_seed_params(const double* __restrict__ p, const double* __restrict__ col,
                              const double* __restrict__ scale, int64_t n, double fixed_ls,
                              double opacity_logit, float* __restrict__ params, int64_t pitch) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ls = fixed_ls;
  if (scale) ls = log(fmax(scale[i], 1e-7));
  float v[kParams] = {(float)p[3 * i], (float)p[3 * i + 1], (float)p[3 * i + 2], (float)ls,
                      (float)ls, (float)ls, 1.f, 0.f, 0.f, 0.f, (float)opacity_logit,
                      (float)col[3 * i], (float)col[3 * i + 1], (float)col[3 * i + 2]};
#pragma unroll
  for (int k = 0; k < kParams; ++k) params[k * pitch + i] = v[k];
}

}  // namespace

void knn_mean_dev(const double* host_pts, const double* pts, int64_t n, int k, double* out,
                  SortScratch& ss, cudaStream_t st) {
  if (n <= 0) return;
  if (k < 1 || k > kMaxK) fail(kInvalidArgument, "knn: k must be in [1, 16]");
  const double* h = host_pts;
  double lo[3] = {h[0], h[1], h[2]}, hi[3] = {h[0], h[1], h[2]};
  for (int64_t i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) {
      lo[c] = std::min(lo[c], h[3 * i + c]);
      hi[c] = std::max(hi[c], h[3 * i + c]);
    }
  double ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  double diag = std::sqrt(ext[0] * ext[0] + ext[1] * ext[1] + ext[2] * ext[2]);
  if (!(diag > 0)) diag = 1.0;
  // surface-like clouds: spacing ~ sqrt(area / n); aim for a few points per cell
  double area = std::max({ext[0] * ext[1], ext[1] * ext[2], ext[0] * ext[2], diag * diag * 1e-6});
  double cell = std::max(2.0 * std::sqrt(area / (double)n), diag * 1e-6);
  Grid g;
  for (int c = 0; c < 3; ++c) {
    g.lo[c] = lo[c];
    g.dims[c] = std::max<int64_t>(1, (int64_t)std::ceil(ext[c] / cell) + 1);
  }
  while ((double)g.dims[0] * g.dims[1] * g.dims[2] > 1.8e19) {
    cell *= 2.0;
    for (int c = 0; c < 3; ++c) g.dims[c] = std::max<int64_t>(1, (int64_t)std::ceil(ext[c] / cell) + 1);
  }
  g.h = cell;
  DevBuf<uint64_t> keys, keys2;
  DevBuf<uint32_t> idx, idx2;
  keys.ensure(n);
  keys2.ensure(n);
  idx.ensure(n);
  idx2.ensure(n);
  unsigned b = (unsigned)((n + 255) / 256);
  k_cell_keys<<<b, 256, 0, st>>>(pts, n, g, keys.get(), idx.get());
  count_launch();
  uint64_t maxkey = (uint64_t)g.dims[0] * g.dims[1] * g.dims[2];
  int bits = 1;
  while (bits < 64 && (uint64_t(1) << bits) < maxkey) ++bits;
  bool alt = radix_sort_pairs<uint64_t>(keys.get(), idx.get(), keys2.get(), idx2.get(), n, 0, bits,
                                        ss, st);
  const uint64_t* sk = alt ? keys2.get() : keys.get();
  const uint32_t* si = alt ? idx2.get() : idx.get();
  k_knn<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(pts, n, g, sk, si, k, out);
  count_launch();
  DSG_CUDA_CHECK(cudaGetLastError());
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
}

void seed_params_dev(const double* pts, const double* colors, const double* scale, int64_t n,
                     double fixed_ls, double opacity_logit, float* params, int64_t pitch,
                     cudaStream_t st) {
  if (n <= 0) return;
  k_seed_params<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pts, colors, scale, n, fixed_ls,
                                                              opacity_logit, params, pitch);
                                                              count_launch();
  DSG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace dsg
