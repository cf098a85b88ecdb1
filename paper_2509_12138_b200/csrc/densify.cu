// Densification and pruning on the device (sm_100a):
// densify_and_prune_impl (trainer.hpp:47-107) + AdamState::remap
// (adam.hpp:36-49) + the stats reset (trainer.hpp:199-201).
//
// Per splat (model order): prune if sigmoid(logit) < prune_opacity; else if
// the mean screen gradient exceeds the threshold, split (max scale above the
// split threshold) or clone; else keep. Output order is the reference's:
// kept splats / first split children / cloned originals in model order,
// then the appended copies and second children in model order. Three
// exclusive scans give every output slot in parallel. The RNG is the
// reference's persistent splitmix64 stream (rng.hpp:8-48): its state
// advances by a constant per draw, and each split consumes exactly 12 draws
// (2 children x 3 normals x 2 uniforms, trainer.hpp:78-79), so split r uses
// draws [12r, 12r+12) after the event's starting state — bit-identical
// children in parallel. Adam moments follow their source (-1 = fresh zeros).
#include <cmath>
#include <cstring>

#include "dsg_internal.h"
#include "raster.h"

namespace dsg {

namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// The k-th draw (0-based) after `state`: splitmix64 adds gamma, then mixes.
__device__ __forceinline__ double uniform_at(uint64_t state, uint64_t k) {
  return (double)(mix64(state + (k + 1) * kGamma) >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ double normal_at(uint64_t state, uint64_t k) {  // rng.hpp:43-48
  double u1 = uniform_at(state, k), u2 = uniform_at(state, k + 1);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

// 0 prune, 1 keep, 2 clone, 3 split (trainer.hpp:68-101)
__global__ void k_densify_classify(const float* __restrict__ P, int64_t pitch, int64_t n,
                                   const double* __restrict__ sg, const int32_t* __restrict__ tc,
                                   double prune_opacity, double grad_thr, double split_thr,
                                   uint8_t* __restrict__ cls, uint32_t* __restrict__ c_main,
                                   uint32_t* __restrict__ c_app, uint32_t* __restrict__ c_split) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double op = 1.0 / (1.0 + exp(-(double)P[10 * pitch + i]));
  uint8_t c = 0;
  if (!(op < prune_opacity)) {
    const double mg = tc[i] > 0 ? sg[i] / tc[i] : 0.0;
    if (mg > grad_thr) {
      const double s = fmax(exp((double)P[3 * pitch + i]),
                            fmax(exp((double)P[4 * pitch + i]), exp((double)P[5 * pitch + i])));
      c = s > split_thr ? 3 : 2;
    } else {
      c = 1;
    }
  }
  cls[i] = c;
  c_main[i] = c ? 1u : 0u;
  c_app[i] = c >= 2 ? 1u : 0u;
  c_split[i] = c == 3 ? 1u : 0u;
}

__global__ void k_densify_scatter(const float* __restrict__ P, const float* __restrict__ M,
                                  const float* __restrict__ V, int64_t pitch, int64_t n,
                                  const uint8_t* __restrict__ cls,
                                  const uint32_t* __restrict__ p_main,
                                  const uint32_t* __restrict__ p_app,
                                  const uint32_t* __restrict__ p_split, uint64_t rng_state,
                                  int64_t n_main, float* __restrict__ P2, float* __restrict__ M2,
                                  float* __restrict__ V2, int64_t pitch2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t c = cls[i];
  if (c == 0) return;
  float p[kParams];
#pragma unroll
  for (int k = 0; k < kParams; ++k) p[k] = P[k * pitch + i];
  const int64_t om = p_main[i];
  const int64_t oa = n_main + (int64_t)p_app[i];
  auto put = [&](int64_t o, const float* q, bool moments) {
#pragma unroll
    for (int k = 0; k < kParams; ++k) {
      P2[k * pitch2 + o] = q[k];
      M2[k * pitch2 + o] = moments ? M[k * pitch + i] : 0.f;
      V2[k * pitch2 + o] = moments ? V[k * pitch + i] : 0.f;
    }
  };
  if (c == 1) {
    put(om, p, true);
  } else if (c == 2) {  // clone: original keeps its moments, the copy is fresh
    put(om, p, true);
    put(oa, p, false);
  } else {  // split into two 0.8x children drawn from the parent's footprint
    double q[4] = {p[6], p[7], p[8], p[9]};
    double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (qn <= 0.0) {
      q[0] = 1; q[1] = q[2] = q[3] = 0;
    } else {
      for (int k = 0; k < 4; ++k) q[k] /= qn;
    }
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    const double s[3] = {exp((double)p[3]), exp((double)p[4]), exp((double)p[5])};
    const double shrink = log(0.8);
    const uint64_t base = 12ull * p_split[i];
    for (int child = 0; child < 2; ++child) {
      const uint64_t k0 = base + 6ull * child;
      const double lx = normal_at(rng_state, k0) * s[0];
      const double ly = normal_at(rng_state, k0 + 2) * s[1];
      const double lz = normal_at(rng_state, k0 + 4) * s[2];
      float cp[kParams];
#pragma unroll
      for (int k = 0; k < kParams; ++k) cp[k] = p[k];
      cp[0] = (float)((double)p[0] + (R[0] * lx + R[1] * ly + R[2] * lz));
      cp[1] = (float)((double)p[1] + (R[3] * lx + R[4] * ly + R[5] * lz));
      cp[2] = (float)((double)p[2] + (R[6] * lx + R[7] * ly + R[8] * lz));
      cp[3] = (float)((double)p[3] + shrink);
      cp[4] = (float)((double)p[4] + shrink);
      cp[5] = (float)((double)p[5] + shrink);
      put(child == 0 ? om : oa, cp, false);
    }
  }
}

__global__ void k_mu_bounds(const float* __restrict__ P, int64_t pitch, int64_t n, int* out) {
  // out[0..2] = min, out[3..5] = max (float atomics via ordered ints)
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float v = P[c * pitch + i];
    const int iv = __float_as_int(v);
    const int key = iv >= 0 ? iv : iv ^ 0x7fffffff;  // monotone int key
    atomicMin(out + c, key);
    atomicMax(out + 3 + c, key);
  }
}

inline unsigned nb(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + 255) / 256); }

}  // namespace

DensifyResult densify_dev(ModelDev& m, ModelDev& spare, DensifyScratch& ds, double prune_opacity,
                          double grad_thr,
                          double split_thr_cfg, uint64_t& rng_state, ScanScratch& sc,
                          cudaStream_t st) {
  DensifyResult r;
  const int64_t n = m.n;
  r.before = n;
  // split threshold: 2% of the model's AABB diagonal when not configured
  double split_thr = split_thr_cfg;
  if (split_thr <= 0.0) {
    double diag = 0.0;
    if (n > 0) {
      DevBuf<int>& b = ds.box;
      b.ensure(6);
      int init[6] = {0x7fffffff, 0x7fffffff, 0x7fffffff, (int)0x80000000, (int)0x80000000,
                     (int)0x80000000};
      DSG_CUDA_CHECK(cudaMemcpyAsync(b.get(), init, sizeof init, cudaMemcpyHostToDevice, st));
      k_mu_bounds<<<nb(n), 256, 0, st>>>(m.params.get(), m.cap, n, b.get());
      count_launch();
      int h[6];
      DSG_CUDA_CHECK(cudaMemcpyAsync(h, b.get(), sizeof h, cudaMemcpyDeviceToHost, st));
      DSG_CUDA_CHECK(cudaStreamSynchronize(st));
      double lo[3], hi[3];
      for (int c = 0; c < 3; ++c) {
        int a = h[c], z = h[3 + c];
        a = a >= 0 ? a : a ^ 0x7fffffff;
        z = z >= 0 ? z : z ^ 0x7fffffff;
        float fa, fz;
        memcpy(&fa, &a, 4);
        memcpy(&fz, &z, 4);
        lo[c] = fa;
        hi[c] = fz;
      }
      diag = std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                       (hi[2] - lo[2]) * (hi[2] - lo[2]));
    }
    split_thr = 0.02 * diag;
  }
  DevBuf<uint8_t>& cls = ds.cls;
  DevBuf<uint32_t>&cm = ds.cm, &ca = ds.ca, &cs = ds.cs;
  cls.ensure(std::max<int64_t>(n, 1));
  cm.ensure(n + 1);
  ca.ensure(n + 1);
  cs.ensure(n + 1);
  k_densify_classify<<<nb(n), 256, 0, st>>>(m.params.get(), m.cap, n, m.stat_norm.get(),
                                            m.stat_count.get(), prune_opacity, grad_thr, split_thr,
                                            cls.get(), cm.get(), ca.get(), cs.get());
  count_launch();
  exclusive_scan_u32(cm.get(), cm.get(), n, sc, st);
  exclusive_scan_u32(ca.get(), ca.get(), n, sc, st);
  exclusive_scan_u32(cs.get(), cs.get(), n, sc, st);
  uint32_t tot[3];
  DSG_CUDA_CHECK(cudaMemcpyAsync(&tot[0], cm.get() + n, 4, cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaMemcpyAsync(&tot[1], ca.get() + n, 4, cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaMemcpyAsync(&tot[2], cs.get() + n, 4, cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  const int64_t n_main = tot[0], n_new = (int64_t)tot[0] + tot[1];
  spare.reserve(std::max<int64_t>(n_new, 1));
  k_densify_scatter<<<nb(n), 256, 0, st>>>(m.params.get(), m.m.get(), m.v.get(), m.cap, n,
                                           cls.get(), cm.get(), ca.get(), cs.get(), rng_state,
                                           n_main, spare.params.get(), spare.m.get(),
                                           spare.v.get(), spare.cap);
  count_launch();
  DSG_CUDA_CHECK(cudaGetLastError());
  rng_state += 12ull * tot[2] * kGamma;  // the stream consumed 12 draws per split
  // swap model storage; stats restart at zero for the new size (trainer.hpp:201)
  m.params.swap(spare.params);
  m.m.swap(spare.m);
  m.v.swap(spare.v);
  std::swap(m.cap, spare.cap);
  m.grads.ensure(kParams * m.cap);
  m.dmean.ensure(2 * m.cap);
  m.touch.ensure(m.cap);
  m.stat_norm.ensure(m.cap);
  m.stat_count.ensure(m.cap);
  m.n = n_new;
  DSG_CUDA_CHECK(cudaMemsetAsync(m.stat_norm.get(), 0, sizeof(double) * m.cap, st));
  DSG_CUDA_CHECK(cudaMemsetAsync(m.stat_count.get(), 0, sizeof(int32_t) * m.cap, st));
  r.after = n_new;
  r.splits = tot[2];
  return r;
}

}  // namespace dsg
