// K7 screen->3D gradient chain (sm_100a).
//
// Replaces the per-splat chain of backward() (backward.hpp:228-330, with
// quat_rotation_derivative :43-69): folds the K6 (duplicate, sub-tile) slots
// of each splat in fixed tile-then-sub-tile order (deterministic, fp64
// accumulation), then chains dL/d(mean2d, conic, colour, alpha_pre) to
// dL/d(mu, log_scale, raw quaternion, opacity logit, colour). The chain runs
// in `Real` (DSG_CHAIN_REAL, default float: the chain is a few dozen
// well-conditioned products per splat and fp32 keeps it bandwidth-bound);
// the symmetric g_Sigma + g_Sigma^T form keeps rotation gradients of
// isotropic identity-rotation splats exactly 0 in either precision.
#include "dsg_internal.h"
#include "raster.h"
#include "adam_math.cuh"

#ifndef DSG_CHAIN_REAL
#define DSG_CHAIN_REAL float
#endif

namespace dsg {

namespace {

using Real = DSG_CHAIN_REAL;

// d R(q)/d q_k for a unit quaternion (backward.hpp:43-69).
__device__ __forceinline__ void drot(const Real* q, int k, Real* m) {
  const Real w = q[0], x = q[1], y = q[2], z = q[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) m[i] = Real(0.0);
  if (k == 0) {
    m[1] = -2 * z; m[2] = 2 * y; m[3] = 2 * z; m[5] = -2 * x; m[6] = -2 * y; m[7] = 2 * x;
  } else if (k == 1) {
    m[1] = 2 * y; m[2] = 2 * z; m[3] = 2 * y; m[4] = -4 * x; m[5] = -2 * w;
    m[6] = 2 * z; m[7] = 2 * w; m[8] = -4 * x;
  } else if (k == 2) {
    m[0] = -4 * y; m[1] = 2 * x; m[2] = 2 * w; m[3] = 2 * x; m[5] = 2 * z;
    m[6] = -2 * w; m[7] = 2 * z; m[8] = -4 * y;
  } else {
    m[0] = -4 * z; m[1] = -2 * w; m[2] = 2 * x; m[3] = 2 * w; m[4] = -4 * z; m[5] = 2 * y;
    m[6] = 2 * x; m[7] = 2 * y;
  }
}

__device__ __forceinline__ void mm3(const Real* a, const Real* b, Real* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}

#ifndef DSG_CHAIN_MINB
#define DSG_CHAIN_MINB 4  // 4 CTAs/SM (64 regs, 72 B spill): 0.34 vs 0.49 ms unbounded
#endif
#ifndef DSG_CHAIN_PAIRS
#define DSG_CHAIN_PAIRS 0
#endif

// kAdam: the training step's fused form — the splat's gradients go straight
// from registers into the Adam update (adam_math.cuh) instead of through the
// planar gradient store (saves 56 B written + 124 B read per splat).
template <bool kAdam>
__global__ void __launch_bounds__(256, DSG_CHAIN_MINB) k_chain(ChainArgs a, AdamArgs ad) {
  DSG_PDL_ENTRY();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  bool touched = false;
  const uint32_t cnt = a.tcount[i];
  if (cnt) {
    // fold (duplicate, sub-tile) slots in fixed tile-then-sub-tile order
    const uint32_t base = a.dup_base[i];
    for (uint32_t k = 0; k < cnt; ++k) {
      const uint32_t d = base + k;
      uint32_t m = (a.tmask[d >> 2] >> (8 * (d & 3))) & 0xffu;
      if (!m) continue;
      touched = true;
      const float4* pp = reinterpret_cast<const float4*>(a.partials) + (size_t)d * 8 * 2;
      const float* p8 = a.partials + (size_t)a.n_dup * 64 + (size_t)d * 8;
#if DSG_CHAIN_PAIRS
      // two rows per round trip (both loads issued before either is summed;
      // the sums stay in sub-tile order)
      while (m) {
        const int w = __ffs(m) - 1;
        m &= m - 1;
        const bool two = m != 0;
        const int w2 = two ? __ffs(m) - 1 : w;
        if (two) m &= m - 1;
        const float4 q0 = __ldg(pp + 2 * w), q1 = __ldg(pp + 2 * w + 1);
        const float e8 = __ldg(p8 + w);
        float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
        float f8 = 0.f;
        if (two) {
          r0 = __ldg(pp + 2 * w2);
          r1 = __ldg(pp + 2 * w2 + 1);
          f8 = __ldg(p8 + w2);
        }
        acc[0] += q0.x;
        acc[1] += q0.y;
        acc[2] += q0.z;
        acc[3] += q0.w;
        acc[4] += q1.x;
        acc[5] += q1.y;
        acc[6] += q1.z;
        acc[7] += q1.w;
        acc[8] += e8;
        if (two) {
          acc[0] += r0.x;
          acc[1] += r0.y;
          acc[2] += r0.z;
          acc[3] += r0.w;
          acc[4] += r1.x;
          acc[5] += r1.y;
          acc[6] += r1.z;
          acc[7] += r1.w;
          acc[8] += f8;
        }
      }
#else
      while (m) {
        const int w = __ffs(m) - 1;
        m &= m - 1;
        const float4 q0 = pp[2 * w], q1 = pp[2 * w + 1];
        acc[0] += q0.x;
        acc[1] += q0.y;
        acc[2] += q0.z;
        acc[3] += q0.w;
        acc[4] += q1.x;
        acc[5] += q1.y;
        acc[6] += q1.z;
        acc[7] += q1.w;
        acc[8] += p8[w];
      }
#endif
    }
  }
  float* G = a.grads;
  const int64_t P = a.pitch;
  if (!touched) {
    if constexpr (kAdam) {
      adam_splat(ad, i, [](int) { return 0.f; }, false, 0.f, 0.f);
    } else {
#pragma unroll
      for (int k = 0; k < kParams; ++k) G[k * P + i] = 0.f;
      a.dmean[i] = 0.f;
      a.dmean[P + i] = 0.f;
      a.touch[i] = 0;
    }
    return;
  }
  Real p[kParams];
#pragma unroll
  for (int k = 0; k < kParams; ++k) p[k] = (Real)a.params[k * P + i];
  const CamDev& c = a.cam;
  Real cR[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) cR[k] = (Real)a.cam.R[k];
  const Real gmx = (Real)acc[0], gmy = (Real)acc[1];
  const Real gca = (Real)acc[2], gcb = (Real)acc[3], gcd = (Real)acc[4];  // g_inv_cov: a, b (= c), d
  // recompute projection geometry (identical math to try_project)
  Real d0 = (Real)((double)a.params[0 * P + i] - c.pos[0]), d1 = (Real)((double)a.params[1 * P + i] - c.pos[1]),
       d2 = (Real)((double)a.params[2 * P + i] - c.pos[2]);
  Real tx = cR[0] * d0 + cR[1] * d1 + cR[2] * d2;
  Real ty = cR[3] * d0 + cR[4] * d1 + cR[5] * d2;
  Real tz = cR[6] * d0 + cR[7] * d1 + cR[8] * d2;
  const Real f = (Real)c.f;
  Real iz = Real(1.0) / tz, iz2 = iz * iz;
  Real j00 = f * iz, j02 = -f * tx * iz2, j11 = -f * iz, j12 = f * ty * iz2;
  Real qr[4] = {p[6], p[7], p[8], p[9]};
  Real qnorm = sqrt(qr[0] * qr[0] + qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3]);
  Real qn[4];
  if (qnorm <= Real(0.0)) {
    qn[0] = 1; qn[1] = qn[2] = qn[3] = 0;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) qn[k] = qr[k] / qnorm;
  }
  Real Rq[9];
  {
    Real w = qn[0], x = qn[1], y = qn[2], z = qn[3];
    Rq[0] = 1 - 2 * (y * y + z * z); Rq[1] = 2 * (x * y - w * z); Rq[2] = 2 * (x * z + w * y);
    Rq[3] = 2 * (x * y + w * z); Rq[4] = 1 - 2 * (x * x + z * z); Rq[5] = 2 * (y * z - w * x);
    Rq[6] = 2 * (x * z - w * y); Rq[7] = 2 * (y * z + w * x); Rq[8] = 1 - 2 * (x * x + y * y);
  }
  Real sc[3] = {exp(p[3]), exp(p[4]), exp(p[5])};
  Real S[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int s = r; s < 3; ++s) {
      Real v = Rq[3 * r] * sc[0] * sc[0] * Rq[3 * s] + Rq[3 * r + 1] * sc[1] * sc[1] * Rq[3 * s + 1] +
                 Rq[3 * r + 2] * sc[2] * sc[2] * Rq[3 * s + 2];
      S[3 * r + s] = v;
      S[3 * s + r] = v;
    }
  Real RT[9] = {cR[0], cR[3], cR[6], cR[1], cR[4], cR[7], cR[2], cR[5], cR[8]};
  Real RS[9], Sc[9];
  mm3(cR, S, RS);
  mm3(RS, RT, Sc);
  // 2D conic from the same geometry
  Real a00 = j00 * Sc[0] + j02 * Sc[6], a01 = j00 * Sc[1] + j02 * Sc[7];
  Real a02 = j00 * Sc[2] + j02 * Sc[8];
  Real b11 = j11 * Sc[4] + j12 * Sc[7], b12 = j11 * Sc[5] + j12 * Sc[8];
  Real cxx = a00 * j00 + a02 * j02 + (Real)kCovDilation;
  Real cxy = a01 * j11 + a02 * j12;
  Real cyy = b11 * j11 + b12 * j12 + (Real)kCovDilation;
  Real det = cxx * cyy - cxy * cxy;
  Real mxx = cyy / det, mxy = -cxy / det, myy = cxx / det;
  Real op = Real(1.0) / (Real(1.0) + exp(-p[10]));

  // dL/dcov2d = -M gM M (backward.hpp:252-261), gM = [[a, b], [b, d]]
  Real t1a = mxx * gca + mxy * gcb, t1b = mxx * gcb + mxy * gcd;
  Real t1c = mxy * gca + myy * gcb, t1d = mxy * gcb + myy * gcd;
  Real ga = -(t1a * mxx + t1b * mxy);
  Real gb = -(t1a * mxy + t1b * myy);
  Real gc = -(t1c * mxx + t1d * mxy);
  Real gd = -(t1c * mxy + t1d * myy);
  // g_sigma_cam = J^T g_cov J
  Real J0[3] = {j00, Real(0.0), j02}, J1[3] = {Real(0.0), j11, j12};
  Real gSc[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int s = 0; s < 3; ++s)
      gSc[3 * r + s] = J0[r] * (ga * J0[s] + gb * J1[s]) + J1[r] * (gc * J0[s] + gd * J1[s]);
  // g_J = (g_cov + g_cov^T) J sigma_cam
  Real sj0[3], sj1[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    sj0[r] = Sc[3 * r] * J0[0] + Sc[3 * r + 1] * J0[1] + Sc[3 * r + 2] * J0[2];
    sj1[r] = Sc[3 * r] * J1[0] + Sc[3 * r + 1] * J1[1] + Sc[3 * r + 2] * J1[2];
  }
  Real gJ0[3], gJ1[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    gJ0[r] = sj0[r] * (Real(2.0) * ga) + sj1[r] * (gb + gc);
    gJ1[r] = sj0[r] * (gb + gc) + sj1[r] * (Real(2.0) * gd);
  }
  Real gtx = gmx * j00;
  Real gty = gmy * j11;
  Real gtz = gmx * (-f * tx * iz2) + gmy * (f * ty * iz2);
  gtx += gJ0[2] * (-f * iz2);
  gty += gJ1[2] * (f * iz2);
  gtz += gJ0[0] * (-f * iz2) + gJ0[2] * (Real(2.0) * f * tx * iz2 * iz) + gJ1[1] * (f * iz2) +
         gJ1[2] * (-Real(2.0) * f * ty * iz2 * iz);
  Real gmu0 = cR[0] * gtx + cR[3] * gty + cR[6] * gtz;
  Real gmu1 = cR[1] * gtx + cR[4] * gty + cR[7] * gtz;
  Real gmu2 = cR[2] * gtx + cR[5] * gty + cR[8] * gtz;
  // g_Sigma = R^T gSc R; g_M3 = (g_Sigma + g_Sigma^T) M3
  Real tmp[9], gS[9];
  mm3(RT, gSc, tmp);
  mm3(tmp, cR, gS);
  Real gsym[9], M3[9], gM3[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      gsym[3 * r + s] = gS[3 * r + s] + gS[3 * s + r];
      M3[3 * r + s] = Rq[3 * r + s] * sc[s];
    }
  mm3(gsym, M3, gM3);
  Real gls[3];
#pragma unroll
  for (int s = 0; s < 3; ++s)
    gls[s] = (gM3[s] * Rq[s] + gM3[3 + s] * Rq[3 + s] + gM3[6 + s] * Rq[6 + s]) * sc[s];
  Real gR[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int s = 0; s < 3; ++s) gR[3 * r + s] = gM3[3 * r + s] * sc[s];
  Real gqn[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Real dr[9];
    drot(qn, k, dr);
    Real v = Real(0.0);
#pragma unroll
    for (int e = 0; e < 9; ++e) v += gR[e] * dr[e];
    gqn[k] = v;
  }
  Real dot = gqn[0] * qn[0] + gqn[1] * qn[1] + gqn[2] * qn[2] + gqn[3] * qn[3];
  float g[kParams];
  g[0] = (float)gmu0;
  g[1] = (float)gmu1;
  g[2] = (float)gmu2;
  g[3] = (float)gls[0];
  g[4] = (float)gls[1];
  g[5] = (float)gls[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) g[6 + k] = (float)((gqn[k] - dot * qn[k]) / qnorm);
  g[10] = (float)(acc[8] * op * (Real(1.0) - op));
  g[11] = (float)acc[5];
  g[12] = (float)acc[6];
  g[13] = (float)acc[7];
  if constexpr (kAdam) {
    adam_splat(ad, i, [&](int k) { return g[k]; }, true, (float)gmx, (float)gmy);
  } else {
#pragma unroll
    for (int k = 0; k < kParams; ++k) G[k * P + i] = g[k];
    a.dmean[i] = (float)gmx;
    a.dmean[P + i] = (float)gmy;
    a.touch[i] = 1;
  }
}

}  // namespace

void chain_3d(const ChainArgs& a, cudaStream_t st) {
  if (a.n == 0) return;
  pdl_launch(k_chain<false>, (unsigned)((a.n + 255) / 256), 256, 0, st, a, AdamArgs{});
  count_launch();
  DSG_CUDA_CHECK(cudaGetLastError());
}

void chain_adam(const ChainArgs& a, const AdamArgs& ad, cudaStream_t st) {
  if (a.n == 0) return;
  pdl_launch(k_chain<true>, (unsigned)((a.n + 255) / 256), 256, 0, st, a, ad);
  count_launch();
  DSG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace dsg
