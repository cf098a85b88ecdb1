// Shared device/host helpers for the dsplat-b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

namespace dsg {

constexpr int kTile = 16;             // internal tile edge (results are tile-size independent,
                                      // render.hpp:157-159 "tiling is a scheduling detail")
constexpr int kTilePx = kTile * kTile;
constexpr int kParams = 14;           // adam.hpp:23
constexpr double kAlphaMax = 0.999;   // render.hpp:18
constexpr double kCovDilation = 0.3;  // projection.hpp:13

// Per-view camera constants, precomputed on the host exactly as the
// reference computes them (camera.hpp:40-62), passed by value to kernels.
struct CamDev {
  double R[9];     // world_to_camera_rotation rows (r, u, f)
  double pos[3];
  double f;        // focal_px
  double half_w;   // 0.5 * width
  double half_h;   // 0.5 * height
  double near_plane;
  int width, height;
  int tiles_x, tiles_y;
  int band_ty0, band_ty1;  // tile rows binned/blended: [band_ty0, band_ty1) (full image by default)
};

// Render-config constants as the kernels use them.
struct RenderDev {
  double sigma_cutoff;
  double sigma_sq;       // sigma_cutoff * sigma_cutoff (render.hpp:175)
  double alpha_cutoff;
  double floor_T;
  float bg[3];
  double bg64[3];
  float sigma_sq_f, alpha_cutoff_f, floor_T_f;
};

// --- exact fp64 arithmetic: no FMA contraction, so device results equal the
// reference's x86-64 (SSE2, unfused) evaluation bit-for-bit. -----------------
__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dd(double a, double b) { return __ddiv_rn(a, b); }

// static_cast<int>(double) as the x86-64 reference executes it (cvttsd2si):
// truncation toward zero, INT_MIN for NaN / out-of-range inputs.
__host__ __device__ __forceinline__ int to_int_x86(double v) {
  if (!(v > -2147483649.0 && v < 2147483648.0)) return INT_MIN;
  return static_cast<int>(v);
}

// Exact fp64 projection of one Gaussian (projection.hpp:24-57 with the
// prepare_splats cull/rect of render.hpp:67-87). Returns false when culled
// by the near plane. Shared by preprocess and the blend guard band so both
// see identical values.
struct Proj64 {
  double mx, my;          // mean2d
  double cxx, cxy, cyy;   // cov2d (dilated)
  double depth;
};

__device__ __forceinline__ void quat_rot64(double w, double x, double y, double z, double* r) {
  r[0] = ds(1.0, dm(2.0, da(dm(y, y), dm(z, z))));
  r[1] = dm(2.0, ds(dm(x, y), dm(w, z)));
  r[2] = dm(2.0, da(dm(x, z), dm(w, y)));
  r[3] = dm(2.0, da(dm(x, y), dm(w, z)));
  r[4] = ds(1.0, dm(2.0, da(dm(x, x), dm(z, z))));
  r[5] = dm(2.0, ds(dm(y, z), dm(w, x)));
  r[6] = dm(2.0, ds(dm(x, z), dm(w, y)));
  r[7] = dm(2.0, da(dm(y, z), dm(w, x)));
  r[8] = ds(1.0, dm(2.0, da(dm(x, x), dm(y, y))));
}

// 3x3 row-major product accumulated from zero (math.hpp:89-95).
__device__ __forceinline__ void mat_mul64(const double* a, const double* b, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = dm(a[3 * i], b[j]);
      s = da(s, dm(a[3 * i + 1], b[3 + j]));
      s = da(s, dm(a[3 * i + 2], b[6 + j]));
      r[3 * i + j] = s;
    }
}

// Camera-space position and 2D EWA covariance in exact fp64. p points at the
// 14 params of one splat as doubles. Returns false if t.z <= near.
__device__ __forceinline__ bool project64(const double* p, const CamDev& c, Proj64& o) {
  double d0 = ds(p[0], c.pos[0]), d1 = ds(p[1], c.pos[1]), d2 = ds(p[2], c.pos[2]);
  double tx = da(da(dm(c.R[0], d0), dm(c.R[1], d1)), dm(c.R[2], d2));
  double ty = da(da(dm(c.R[3], d0), dm(c.R[4], d1)), dm(c.R[5], d2));
  double tz = da(da(dm(c.R[6], d0), dm(c.R[7], d1)), dm(c.R[8], d2));
  if (tz <= c.near_plane) return false;
  double iz = dd(1.0, tz);
  double iz2 = dm(iz, iz);
  double j00 = dm(c.f, iz), j02 = dm(dm(-c.f, tx), iz2);
  double j11 = dm(-c.f, iz), j12 = dm(dm(c.f, ty), iz2);
  // rot.normalized() (math.hpp:57-61)
  double qw = p[6], qx = p[7], qy = p[8], qz = p[9];
  double qn = sqrt(da(da(da(dm(qw, qw), dm(qx, qx)), dm(qy, qy)), dm(qz, qz)));
  if (qn <= 0.0) {
    qw = 1.0; qx = qy = qz = 0.0;
  } else {
    qw = dd(qw, qn); qx = dd(qx, qn); qy = dd(qy, qn); qz = dd(qz, qn);
  }
  double r[9];
  quat_rot64(qw, qx, qy, qz, r);
  double s2[3] = {exp(dm(2.0, p[3])), exp(dm(2.0, p[4])), exp(dm(2.0, p[5]))};
  double S[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j) {
      double v = dm(dm(r[3 * i], s2[0]), r[3 * j]);
      v = da(v, dm(dm(r[3 * i + 1], s2[1]), r[3 * j + 1]));
      v = da(v, dm(dm(r[3 * i + 2], s2[2]), r[3 * j + 2]));
      S[3 * i + j] = v;
      S[3 * j + i] = v;
    }
  double RT[9] = {c.R[0], c.R[3], c.R[6], c.R[1], c.R[4], c.R[7], c.R[2], c.R[5], c.R[8]};
  double RS[9], Sc[9];
  mat_mul64(c.R, S, RS);
  mat_mul64(RS, RT, Sc);
  double a00 = da(dm(j00, Sc[0]), dm(j02, Sc[6]));
  double a01 = da(dm(j00, Sc[1]), dm(j02, Sc[7]));
  double a02 = da(dm(j00, Sc[2]), dm(j02, Sc[8]));
  double b11 = da(dm(j11, Sc[4]), dm(j12, Sc[7]));
  double b12 = da(dm(j11, Sc[5]), dm(j12, Sc[8]));
  o.cxx = da(da(dm(a00, j00), dm(a02, j02)), kCovDilation);
  o.cxy = da(dm(a01, j11), dm(a02, j12));
  o.cyy = da(da(dm(b11, j11), dm(b12, j12)), kCovDilation);
  o.mx = da(c.half_w, dd(dm(c.f, tx), tz));
  o.my = ds(c.half_h, dd(dm(c.f, ty), tz));
  o.depth = tz;
  return true;
}

__device__ __forceinline__ double sigmoid64(double v) { return dd(1.0, da(1.0, exp(-v))); }

// Outcome of one (pixel, splat) evaluation of splat_alpha_at
// (render.hpp:140-154) plus the backward clamp gate (backward.hpp:142).
struct AlphaEval {
  float alpha;   // min(o*g, 0.999)
  float om;      // 1 - alpha, formed so the 0.999 clamp gives exactly 1e-3
  float g;       // gaussian value
  bool gate;     // o*g <= 0.999 (gradient flows through the clamp)
  float err;     // bound on alpha's relative error (forward's termination bound)
};

}  // namespace dsg

#define DSG_CUDA_CHECK(expr)                                                   \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) ::dsg::throw_cuda(_e, #expr, __FILE__, __LINE__);   \
  } while (0)

namespace dsg {
[[noreturn]] void throw_cuda(cudaError_t e, const char* expr, const char* file, int line);
}

// ---- programmatic dependent launch (sm_90+; used on the per-step path) -----
// Every per-step kernel is launched with programmatic stream serialization
// and starts with DSG_PDL_ENTRY(): it waits for its predecessor grid to
// complete (and its writes to be visible) before touching memory, then lets
// its own successor launch as soon as all of its blocks are resident, so the
// successor's launch and block scheduling overlap this grid's tail instead
// of following it.
#ifndef DSG_NO_PDL
#define DSG_PDL_ENTRY()                                   \
  do {                                                    \
    asm volatile("griddepcontrol.wait;" ::: "memory");    \
    asm volatile("griddepcontrol.launch_dependents;" ::); \
  } while (0)
#else  // A/B builds without PDL
#define DSG_PDL_ENTRY() \
  do {                  \
  } while (0)
#endif

namespace dsg {
void count_launch(int n);
template <class... KArgs, class... Args>
inline void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
#ifndef DSG_NO_PDL
  cfg.numAttrs = 1;
#else
  cfg.numAttrs = 0;
#endif
  DSG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}
}  // namespace dsg
