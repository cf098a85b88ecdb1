// K7 screen->3D gradient chain and K9 fused Adam (sm_100a).
//
// K7 replaces the per-splat chain of backward() (backward.hpp:228-330, with
// quat_rotation_derivative :43-69): it folds the K6 duplicate slots of each
// splat in tile order (deterministic), then chains dL/d(mean2d, conic,
// colour, alpha_pre) to dL/d(mu, log_scale, raw quaternion, opacity logit,
// colour) in fp64. The symmetric g_Sigma + g_Sigma^T form is kept so
// rotation gradients of isotropic identity-rotation splats stay exactly 0.
//
// K9 replaces AdamState::step (adam.hpp:55-101) and the densification
// statistics update (gradient.hpp:39-45, trainer.hpp:189-193): one pass over
// the planar fp32 params/grads/moments, quaternion renormalisation and
// log-scale clamp fused in.
#include "dsg_internal.h"
#include "raster.h"

namespace dsg {

namespace {


#ifndef DSG_ADAM_BATCH
#define DSG_ADAM_BATCH 1
#endif
#ifndef DSG_ADAM_MINB
#define DSG_ADAM_MINB 1
#endif
__global__ void __launch_bounds__(256, DSG_ADAM_MINB) k_adam(AdamArgs a) {
  DSG_PDL_ENTRY();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const int64_t P = a.pitch;
  float p[kParams];
#if DSG_ADAM_BATCH
  // the four planes never alias: all loads of a half (7 parameters) are
  // issued before its stores, 28 in flight per thread instead of 3
  const float* __restrict__ G = a.grads;
  float* __restrict__ M = a.m;
  float* __restrict__ V = a.v;
  const float* __restrict__ Q = a.params;
  constexpr int kHalf = kParams / 2;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float g[kHalf], m0[kHalf], v0[kHalf], q[kHalf];
#pragma unroll
    for (int j = 0; j < kHalf; ++j) {
      const int64_t o = (h * kHalf + j) * P + i;
      g[j] = __ldg(G + o);
      m0[j] = M[o];
      v0[j] = V[o];
      q[j] = __ldg(Q + o);
    }
#pragma unroll
    for (int j = 0; j < kHalf; ++j) {
      const int k = h * kHalf + j;
      const int grp = k < 3 ? 0 : (k < 6 ? 1 : (k < 10 ? 2 : (k == 10 ? 3 : 4)));
      const int64_t o = k * P + i;
      const float m = a.b1 * m0[j] + a.omb1 * g[j];
      const float v = a.b2 * v0[j] + a.omb2 * g[j] * g[j];
      M[o] = m;
      V[o] = v;
      const float mh = m * a.inv_bc1, vh = v * a.inv_bc2;
      p[k] = q[j] - a.lr[grp] * mh / (sqrtf(vh) + a.eps);
    }
  }
#else
#pragma unroll
  for (int k = 0; k < kParams; ++k) {
    const int grp = k < 3 ? 0 : (k < 6 ? 1 : (k < 10 ? 2 : (k == 10 ? 3 : 4)));
    const int64_t o = k * P + i;
    float g = a.grads[o];
    float m = a.b1 * a.m[o] + a.omb1 * g;
    float v = a.b2 * a.v[o] + a.omb2 * g * g;
    a.m[o] = m;
    a.v[o] = v;
    float mh = m * a.inv_bc1, vh = v * a.inv_bc2;
    p[k] = a.params[o] - a.lr[grp] * mh / (sqrtf(vh) + a.eps);
  }
#endif
  // normalize_rotation (gaussian.hpp:31, math.hpp:57-61) and clamp_scale (:32-37)
  float qn = sqrtf(p[6] * p[6] + p[7] * p[7] + p[8] * p[8] + p[9] * p[9]);
  if (qn <= 0.f) {
    p[6] = 1.f; p[7] = p[8] = p[9] = 0.f;
  } else {
#pragma unroll
    for (int k = 6; k < 10; ++k) p[k] = p[k] / qn;
  }
#pragma unroll
  for (int k = 3; k < 6; ++k) p[k] = fminf(fmaxf(p[k], a.ls_lo), a.ls_hi);
#pragma unroll
  for (int k = 0; k < kParams; ++k) a.params[k * P + i] = p[k];
  if (a.accumulate_stats && a.touch[i] > 0) {
    const double dx = a.dmean[i], dy = a.dmean[P + i];
    a.stat_norm[i] += sqrt(dx * dx + dy * dy);  // d_mean2d.norm() (trainer.hpp:189-193)
    a.stat_count[i] += 1;
  }
}

}  // namespace

void adam_update(const AdamArgs& a, cudaStream_t st) {
  if (a.n == 0) return;
  pdl_launch(k_adam, (unsigned)((a.n + 255) / 256), 256, 0, st, a);
  count_launch();
  DSG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace dsg
