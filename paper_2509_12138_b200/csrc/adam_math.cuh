// AdamState::step for one splat (adam.hpp:55-101) with normalize_rotation
// (gaussian.hpp:31, math.hpp:57-61), clamp_scale (:32-37) and the
// densification statistics (trainer.hpp:189-193). Shared by k_adam
// (gradients loaded from the planar store) and the fused chain + Adam kernel
// (gradients still in registers, chain.cu): same expressions, same bits.
#pragma once
#include "raster.h"

namespace dsg {

// grad(k): the splat's k-th gradient; touched / dmx / dmy: whether any pixel
// reached it this step and its screen-space mean gradient (float, as stored).
template <class GradOf>
__device__ __forceinline__ void adam_splat(const AdamArgs& a, int64_t i, GradOf grad,
                                           bool touched, float dmx, float dmy) {
  const int64_t P = a.pitch;
  float p[kParams];
  // the planes never alias: all loads of a half (7 parameters) are issued
  // before its stores, 28 in flight per thread instead of 3
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
      g[j] = grad(h * kHalf + j);
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
  float qn = sqrtf(p[6] * p[6] + p[7] * p[7] + p[8] * p[8] + p[9] * p[9]);
  if (qn <= 0.f) {
    p[6] = 1.f;
    p[7] = p[8] = p[9] = 0.f;
  } else {
#pragma unroll
    for (int k = 6; k < 10; ++k) p[k] = p[k] / qn;
  }
#pragma unroll
  for (int k = 3; k < 6; ++k) p[k] = fminf(fmaxf(p[k], a.ls_lo), a.ls_hi);
  float* __restrict__ W = a.params;
#pragma unroll
  for (int k = 0; k < kParams; ++k) W[k * P + i] = p[k];
  if (a.accumulate_stats && touched) {
    const double dx = dmx, dy = dmy;
    a.stat_norm[i] += sqrt(dx * dx + dy * dy);  // d_mean2d.norm() (trainer.hpp:189-193)
    a.stat_count[i] += 1;
  }
}

}  // namespace dsg
