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

#if 0  // K7 moved to chain.cu (precision-templated); kept here for reference until removed
// d R(q)/d q_k for a unit quaternion (backward.hpp:43-69).
__device__ __forceinline__ void drot(const double* q, int k, double* m) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) m[i] = 0.0;
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

__device__ __forceinline__ void mm3(const double* a, const double* b, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}

__global__ void __launch_bounds__(256) k_chain(ChainArgs a) {
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
      const float* pp = a.partials + (size_t)d * 8 * 9;
      while (m) {
        const int w = __ffs(m) - 1;
        m &= m - 1;
        const float* q = pp + w * 9;
#pragma unroll
        for (int v = 0; v < 9; ++v) acc[v] += q[v];
      }
    }
  }
  float* G = a.grads;
  const int64_t P = a.pitch;
  if (!touched) {
#pragma unroll
    for (int k = 0; k < kParams; ++k) G[k * P + i] = 0.f;
    a.dmean[i] = 0.f;
    a.dmean[P + i] = 0.f;
    a.touch[i] = 0;
    return;
  }
  double p[kParams];
#pragma unroll
  for (int k = 0; k < kParams; ++k) p[k] = (double)a.params[k * P + i];
  const CamDev& c = a.cam;
  const double gmx = acc[0], gmy = acc[1];
  const double gca = acc[2], gcb = acc[3], gcd = acc[4];  // g_inv_cov: a, b (= c), d
  // recompute projection geometry (identical math to try_project)
  double d0 = p[0] - c.pos[0], d1 = p[1] - c.pos[1], d2 = p[2] - c.pos[2];
  double tx = c.R[0] * d0 + c.R[1] * d1 + c.R[2] * d2;
  double ty = c.R[3] * d0 + c.R[4] * d1 + c.R[5] * d2;
  double tz = c.R[6] * d0 + c.R[7] * d1 + c.R[8] * d2;
  const double f = c.f;
  double iz = 1.0 / tz, iz2 = iz * iz;
  double j00 = f * iz, j02 = -f * tx * iz2, j11 = -f * iz, j12 = f * ty * iz2;
  double qr[4] = {p[6], p[7], p[8], p[9]};
  double qnorm = sqrt(qr[0] * qr[0] + qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3]);
  double qn[4];
  if (qnorm <= 0.0) {
    qn[0] = 1; qn[1] = qn[2] = qn[3] = 0;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) qn[k] = qr[k] / qnorm;
  }
  double Rq[9];
  {
    double w = qn[0], x = qn[1], y = qn[2], z = qn[3];
    Rq[0] = 1 - 2 * (y * y + z * z); Rq[1] = 2 * (x * y - w * z); Rq[2] = 2 * (x * z + w * y);
    Rq[3] = 2 * (x * y + w * z); Rq[4] = 1 - 2 * (x * x + z * z); Rq[5] = 2 * (y * z - w * x);
    Rq[6] = 2 * (x * z - w * y); Rq[7] = 2 * (y * z + w * x); Rq[8] = 1 - 2 * (x * x + y * y);
  }
  double sc[3] = {exp(p[3]), exp(p[4]), exp(p[5])};
  double S[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int s = r; s < 3; ++s) {
      double v = Rq[3 * r] * sc[0] * sc[0] * Rq[3 * s] + Rq[3 * r + 1] * sc[1] * sc[1] * Rq[3 * s + 1] +
                 Rq[3 * r + 2] * sc[2] * sc[2] * Rq[3 * s + 2];
      S[3 * r + s] = v;
      S[3 * s + r] = v;
    }
  double RT[9] = {c.R[0], c.R[3], c.R[6], c.R[1], c.R[4], c.R[7], c.R[2], c.R[5], c.R[8]};
  double RS[9], Sc[9];
  mm3(c.R, S, RS);
  mm3(RS, RT, Sc);
  // 2D conic from the same geometry
  double a00 = j00 * Sc[0] + j02 * Sc[6], a01 = j00 * Sc[1] + j02 * Sc[7];
  double a02 = j00 * Sc[2] + j02 * Sc[8];
  double b11 = j11 * Sc[4] + j12 * Sc[7], b12 = j11 * Sc[5] + j12 * Sc[8];
  double cxx = a00 * j00 + a02 * j02 + kCovDilation;
  double cxy = a01 * j11 + a02 * j12;
  double cyy = b11 * j11 + b12 * j12 + kCovDilation;
  double det = cxx * cyy - cxy * cxy;
  double mxx = cyy / det, mxy = -cxy / det, myy = cxx / det;
  double op = 1.0 / (1.0 + exp(-p[10]));

  // dL/dcov2d = -M gM M (backward.hpp:252-261), gM = [[a, b], [b, d]]
  double t1a = mxx * gca + mxy * gcb, t1b = mxx * gcb + mxy * gcd;
  double t1c = mxy * gca + myy * gcb, t1d = mxy * gcb + myy * gcd;
  double ga = -(t1a * mxx + t1b * mxy);
  double gb = -(t1a * mxy + t1b * myy);
  double gc = -(t1c * mxx + t1d * mxy);
  double gd = -(t1c * mxy + t1d * myy);
  // g_sigma_cam = J^T g_cov J
  double J0[3] = {j00, 0.0, j02}, J1[3] = {0.0, j11, j12};
  double gSc[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int s = 0; s < 3; ++s)
      gSc[3 * r + s] = J0[r] * (ga * J0[s] + gb * J1[s]) + J1[r] * (gc * J0[s] + gd * J1[s]);
  // g_J = (g_cov + g_cov^T) J sigma_cam
  double sj0[3], sj1[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    sj0[r] = Sc[3 * r] * J0[0] + Sc[3 * r + 1] * J0[1] + Sc[3 * r + 2] * J0[2];
    sj1[r] = Sc[3 * r] * J1[0] + Sc[3 * r + 1] * J1[1] + Sc[3 * r + 2] * J1[2];
  }
  double gJ0[3], gJ1[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    gJ0[r] = sj0[r] * (2.0 * ga) + sj1[r] * (gb + gc);
    gJ1[r] = sj0[r] * (gb + gc) + sj1[r] * (2.0 * gd);
  }
  double gtx = gmx * j00;
  double gty = gmy * j11;
  double gtz = gmx * (-f * tx * iz2) + gmy * (f * ty * iz2);
  gtx += gJ0[2] * (-f * iz2);
  gty += gJ1[2] * (f * iz2);
  gtz += gJ0[0] * (-f * iz2) + gJ0[2] * (2.0 * f * tx * iz2 * iz) + gJ1[1] * (f * iz2) +
         gJ1[2] * (-2.0 * f * ty * iz2 * iz);
  double gmu0 = c.R[0] * gtx + c.R[3] * gty + c.R[6] * gtz;
  double gmu1 = c.R[1] * gtx + c.R[4] * gty + c.R[7] * gtz;
  double gmu2 = c.R[2] * gtx + c.R[5] * gty + c.R[8] * gtz;
  // g_Sigma = R^T gSc R; g_M3 = (g_Sigma + g_Sigma^T) M3
  double tmp[9], gS[9];
  mm3(RT, gSc, tmp);
  mm3(tmp, c.R, gS);
  double gsym[9], M3[9], gM3[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      gsym[3 * r + s] = gS[3 * r + s] + gS[3 * s + r];
      M3[3 * r + s] = Rq[3 * r + s] * sc[s];
    }
  mm3(gsym, M3, gM3);
  double gls[3];
#pragma unroll
  for (int s = 0; s < 3; ++s)
    gls[s] = (gM3[s] * Rq[s] + gM3[3 + s] * Rq[3 + s] + gM3[6 + s] * Rq[6 + s]) * sc[s];
  double gR[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int s = 0; s < 3; ++s) gR[3 * r + s] = gM3[3 * r + s] * sc[s];
  double gqn[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double dr[9];
    drot(qn, k, dr);
    double v = 0.0;
#pragma unroll
    for (int e = 0; e < 9; ++e) v += gR[e] * dr[e];
    gqn[k] = v;
  }
  double dot = gqn[0] * qn[0] + gqn[1] * qn[1] + gqn[2] * qn[2] + gqn[3] * qn[3];
  G[0 * P + i] = (float)gmu0;
  G[1 * P + i] = (float)gmu1;
  G[2 * P + i] = (float)gmu2;
  G[3 * P + i] = (float)gls[0];
  G[4 * P + i] = (float)gls[1];
  G[5 * P + i] = (float)gls[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) G[(6 + k) * P + i] = (float)((gqn[k] - dot * qn[k]) / qnorm);
  G[10 * P + i] = (float)(acc[8] * op * (1.0 - op));
  G[11 * P + i] = (float)acc[5];
  G[12 * P + i] = (float)acc[6];
  G[13 * P + i] = (float)acc[7];
  a.dmean[i] = (float)gmx;
  a.dmean[P + i] = (float)gmy;
  a.touch[i] = 1;
}
#endif

__global__ void __launch_bounds__(256) k_adam(AdamArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const int64_t P = a.pitch;
  float p[kParams];
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
    float dx = a.dmean[i], dy = a.dmean[P + i];
    a.stat_norm[i] += sqrtf(dx * dx + dy * dy);
    a.stat_count[i] += 1;
  }
}

}  // namespace

void adam_update(const AdamArgs& a, cudaStream_t st) {
  if (a.n == 0) return;
  k_adam<<<(unsigned)((a.n + 255) / 256), 256, 0, st>>>(a);
  count_launch();
  DSG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace dsg
