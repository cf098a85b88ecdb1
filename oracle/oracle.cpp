// TEST INFRASTRUCTURE ONLY — the CPU oracle.
//
// A from-scratch fp64 restatement of the reference algorithm for the hot
// path (/root/reference/proj/include/dsplat/*.hpp), written as flat C-style
// loops over the oracle ABI's AoS arrays (orc_abi.h). Every function cites
// the reference file:line it restates and keeps the reference's
// floating-point evaluation order, so on the same inputs it reproduces the
// reference bit-for-bit; tests/test_oracle_pin.py checks that against
// oracle/_ref (the reference headers compiled unchanged) and
// tests/test_golden.py against the reference-generated fixtures in
// tests/golden/golden.npz (tests/golden/make_golden.py).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// load this library. The product (paper_2509_12138_b200/libdsg.so) never
// links or calls it.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "orc_abi.h"

namespace {

// ---- errors (error.hpp:10-69) ---------------------------------------------
enum Code {
  kBehindCamera = 0, kInvalidRig, kUnknownKind, kIsovalueOutOfRange, kEmptyCloud,
  kDimensionMismatch, kTooSmall, kEmptyBand, kEmptyInterior, kMismatchedCounts, kNoViews,
  kStaleForward, kIoError, kMalformedFile, kWorkerFailure, kTimeout, kManifestMismatch,
  kMissingBaseline, kInvalidArgument
};
const char* kCodeNames[] = {"BehindCamera", "InvalidRig", "UnknownKind", "IsovalueOutOfRange",
                            "EmptyCloud", "DimensionMismatch", "TooSmall", "EmptyBand",
                            "EmptyInterior", "MismatchedCounts", "NoViews", "StaleForward",
                            "IoError", "MalformedFile", "WorkerFailure", "Timeout",
                            "ManifestMismatch", "MissingBaseline", "InvalidArgument"};
struct Fail {
  int code;
  std::string msg;
};
thread_local std::string g_err;
[[noreturn]] void fail(int code, const char* msg) { throw Fail{code, msg}; }
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Fail& e) {
    g_err = std::string(kCodeNames[e.code]) + ": " + e.msg;
    return e.code + 1;
  }
}

// ---- small vector helpers (math.hpp:14-171) -------------------------------
struct V3 {
  double x, y, z;
};
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline double dot3(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross3(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double len3(V3 a) { return std::sqrt(dot3(a, a)); }
inline V3 unit3(V3 a) {  // Vec3::normalized, math.hpp:39-42
  double n = len3(a);
  return n > 0.0 ? V3{a.x / n, a.y / n, a.z / n} : V3{0.0, 0.0, 0.0};
}
// 3x3 row-major product accumulated from zero (math.hpp:89-95).
inline void mat_mul(const double* a, const double* b, double* r) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += a[3 * i + k] * b[3 * k + j];
      r[3 * i + j] = s;
    }
}
inline void mat_T(const double* a, double* r) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[3 * i + j] = a[3 * j + i];
}
inline double sigmoid(double v) { return 1.0 / (1.0 + std::exp(-v)); }

// static_cast<int>(double) as the x86-64 reference build executes it
// (cvttsd2si): truncation, and INT_MIN for NaN or out-of-range values.
inline int to_int_x86(double v) {
  if (!(v > -2147483649.0 && v < 2147483648.0)) return std::numeric_limits<int>::min();
  return static_cast<int>(v);
}

// Unit quaternion (w,x,y,z) -> rotation matrix (math.hpp:133-146).
inline void quat_rot(double w, double x, double y, double z, double* r) {
  r[0] = 1 - 2 * (y * y + z * z);
  r[1] = 2 * (x * y - w * z);
  r[2] = 2 * (x * z + w * y);
  r[3] = 2 * (x * y + w * z);
  r[4] = 1 - 2 * (x * x + z * z);
  r[5] = 2 * (y * z - w * x);
  r[6] = 2 * (x * z - w * y);
  r[7] = 2 * (y * z + w * x);
  r[8] = 1 - 2 * (x * x + y * y);
}

// Quat::normalized (math.hpp:57-61).
inline void quat_unit(const double* q, double* out) {
  double n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  if (n <= 0.0) {
    out[0] = 1.0; out[1] = out[2] = out[3] = 0.0;
    return;
  }
  for (int k = 0; k < 4; ++k) out[k] = q[k] / n;
}

// Sigma = R diag(e^{2s}) R^T (gaussian.hpp:58-72), qn already normalized.
inline void covariance3(const double* ls, const double* qn, double* cov) {
  double r[9];
  quat_rot(qn[0], qn[1], qn[2], qn[3], r);
  double s2[3] = {std::exp(2.0 * ls[0]), std::exp(2.0 * ls[1]), std::exp(2.0 * ls[2])};
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j) {
      double v = r[3 * i] * s2[0] * r[3 * j] + r[3 * i + 1] * s2[1] * r[3 * j + 1] +
                 r[3 * i + 2] * s2[2] * r[3 * j + 2];
      cov[3 * i + j] = v;
      cov[3 * j + i] = v;
    }
}

// ---- camera (camera.hpp:16-70) ---------------------------------------------
struct Cam {
  V3 pos, tgt, up;
  double fov, nearp, farp;
  int w, h;
  double R[9];  // world_to_camera_rotation rows (r, u, f), camera.hpp:40-49
  double f;     // focal_px, camera.hpp:56
};

Cam make_cam(const orc_camera* c) {
  Cam k;
  k.pos = {c->position[0], c->position[1], c->position[2]};
  k.tgt = {c->target[0], c->target[1], c->target[2]};
  k.up = {c->up[0], c->up[1], c->up[2]};
  k.fov = c->fov_y;
  k.w = c->width;
  k.h = c->height;
  k.nearp = c->near_plane;
  k.farp = c->far_plane;
  V3 fw = unit3(sub(k.tgt, k.pos));
  V3 rt = unit3(cross3(fw, k.up));
  V3 u = cross3(rt, fw);
  double R[9] = {rt.x, rt.y, rt.z, u.x, u.y, u.z, fw.x, fw.y, fw.z};
  std::memcpy(k.R, R, sizeof R);
  k.f = 0.5 * k.h / std::tan(0.5 * k.fov);
  return k;
}

// Camera::validate (camera.hpp:26-36).
void validate_cam(const Cam& k) {
  if (k.w < 8 || k.h < 8) fail(kInvalidRig, "camera resolution below 8 px");
  if (!(k.fov > 0.0 && k.fov < M_PI)) fail(kInvalidRig, "fov_y outside (0, pi)");
  if (!(k.nearp < k.farp)) fail(kInvalidRig, "near must be < far");
  V3 dir = sub(k.tgt, k.pos);
  if (len3(cross3(dir, k.up)) <= 1e-12 * len3(dir) * len3(k.up))
    fail(kInvalidRig, "up parallel to view direction");
}

inline V3 to_cam_space(const Cam& k, V3 p) {
  V3 d = sub(p, k.pos);
  return {k.R[0] * d.x + k.R[1] * d.y + k.R[2] * d.z, k.R[3] * d.x + k.R[4] * d.y + k.R[5] * d.z,
          k.R[6] * d.x + k.R[7] * d.y + k.R[8] * d.z};
}

// ---- render config (render.hpp:20-35) --------------------------------------
void validate_cfg(const orc_render_cfg* c) {
  if (c->tile_size <= 0 || (c->tile_size & (c->tile_size - 1)) != 0)
    fail(kInvalidArgument, "tile_size must be a positive power of two");
  if (!(c->alpha_cutoff > 0.0 && c->alpha_cutoff < 1.0))
    fail(kInvalidArgument, "alpha_cutoff outside (0, 1)");
  if (!(c->sigma_cutoff >= 1.0 && c->sigma_cutoff <= 6.0))
    fail(kInvalidArgument, "sigma_cutoff outside [1, 6]");
}

const double kAlphaCap = 0.999;   // render.hpp:18
const double kDilation = 0.3;     // projection.hpp:13

// One entry of the compositing list (PreparedSplat, render.hpp:48-57).
struct Splat {
  double mx, my;         // mean2d
  double ixx, ixy, iyy;  // inverse cov2d
  double op;             // sigmoid(opacity_logit)
  double cr, cg, cb;     // color
  double depth;
  int32_t idx;
  int x0, x1, y0, y1;
};

// try_project + prepare_splats (projection.hpp:24-57, render.hpp:62-103).
std::vector<Splat> project_sort(const double* P, int64_t n, const Cam& k,
                                const orc_render_cfg* cfg) {
  std::vector<Splat> out;
  out.reserve(static_cast<size_t>(n));
  double RT[9];
  mat_T(k.R, RT);
  for (int64_t i = 0; i < n; ++i) {
    const double* g = P + 14 * i;
    V3 t = to_cam_space(k, {g[0], g[1], g[2]});
    if (t.z <= k.nearp) continue;
    double iz = 1.0 / t.z, iz2 = iz * iz;
    double j00 = k.f * iz, j02 = -k.f * t.x * iz2;
    double j11 = -k.f * iz, j12 = k.f * t.y * iz2;
    double qn[4], S[9], RS[9], Sc[9];
    quat_unit(g + 6, qn);
    covariance3(g + 3, qn, S);
    mat_mul(k.R, S, RS);
    mat_mul(RS, RT, Sc);
    double a00 = j00 * Sc[0] + j02 * Sc[6];
    double a01 = j00 * Sc[1] + j02 * Sc[7];
    double a02 = j00 * Sc[2] + j02 * Sc[8];
    double b11 = j11 * Sc[4] + j12 * Sc[7];
    double b12 = j11 * Sc[5] + j12 * Sc[8];
    double cxx = a00 * j00 + a02 * j02 + kDilation;
    double cxy = a01 * j11 + a02 * j12;
    double cyy = b11 * j11 + b12 * j12 + kDilation;
    double mx = 0.5 * k.w + k.f * t.x / t.z;
    double my = 0.5 * k.h - k.f * t.y / t.z;
    double rx = cfg->sigma_cutoff * std::sqrt(cxx);
    double ry = cfg->sigma_cutoff * std::sqrt(cyy);
    int x0 = std::max(to_int_x86(std::ceil(mx - rx - 0.5)), 0);
    int x1 = std::min(to_int_x86(std::floor(mx + rx - 0.5)), k.w - 1);
    int y0 = std::max(to_int_x86(std::ceil(my - ry - 0.5)), 0);
    int y1 = std::min(to_int_x86(std::floor(my + ry - 0.5)), k.h - 1);
    if (x0 > x1 || y0 > y1) continue;
    double det = cxx * cyy - cxy * cxy;
    if (det <= 0.0) continue;
    Splat s;
    s.mx = mx;
    s.my = my;
    s.ixx = cyy / det;
    s.ixy = -cxy / det;
    s.iyy = cxx / det;
    s.op = sigmoid(g[10]);
    s.cr = g[11];
    s.cg = g[12];
    s.cb = g[13];
    s.depth = t.z;
    s.idx = static_cast<int32_t>(i);
    s.x0 = x0;
    s.x1 = x1;
    s.y0 = y0;
    s.y1 = y1;
    out.push_back(s);
  }
  std::sort(out.begin(), out.end(), [](const Splat& a, const Splat& b) {
    if (a.depth != b.depth) return a.depth < b.depth;
    return a.idx < b.idx;
  });
  return out;
}

// Tile lists of positions into the sorted list (render.hpp:117-135), stored
// CSR-style: start[t] .. start[t+1].
struct Bins {
  int tx, ty, ts;
  std::vector<int64_t> start;
  std::vector<int32_t> pos;
  int tile_of(int x, int y) const { return (y / ts) * tx + (x / ts); }
};

Bins make_bins(const std::vector<Splat>& s, int w, int h, int ts) {
  Bins b;
  b.ts = ts;
  b.tx = (w + ts - 1) / ts;
  b.ty = (h + ts - 1) / ts;
  size_t nt = static_cast<size_t>(b.tx) * static_cast<size_t>(b.ty);
  std::vector<int64_t> cnt(nt + 1, 0);
  for (const Splat& p : s)
    for (int y = p.y0 / ts; y <= p.y1 / ts; ++y)
      for (int x = p.x0 / ts; x <= p.x1 / ts; ++x) ++cnt[static_cast<size_t>(y * b.tx + x) + 1];
  for (size_t t = 0; t < nt; ++t) cnt[t + 1] += cnt[t];
  b.start = cnt;
  b.pos.assign(static_cast<size_t>(cnt[nt]), 0);
  std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
  for (size_t i = 0; i < s.size(); ++i) {
    const Splat& p = s[i];
    for (int y = p.y0 / ts; y <= p.y1 / ts; ++y)
      for (int x = p.x0 / ts; x <= p.x1 / ts; ++x)
        b.pos[static_cast<size_t>(fill[static_cast<size_t>(y * b.tx + x)]++)] = static_cast<int32_t>(i);
  }
  return b;
}

// splat_alpha_at (render.hpp:140-154).
inline bool alpha_at(const Splat& p, double px, double py, double sig2, double cutoff,
                     double* alpha, double* gauss) {
  double dx = px - p.mx;
  double dy = py - p.my;
  double q = p.ixx * dx * dx + 2.0 * p.ixy * dx * dy + p.iyy * dy * dy;
  if (q > sig2) return false;
  double g = std::exp(-0.5 * q);
  double a = p.op * g;
  if (a > kAlphaCap) a = kAlphaCap;
  if (a < cutoff) return false;
  *alpha = a;
  *gauss = g;
  return true;
}

// ---- SSIM (ssim.hpp:17-121) -------------------------------------------------
const int kWin = 11;
const double kC1 = 0.01 * 0.01;
const double kC2 = 0.03 * 0.03;

const double* ssim_window() {
  static double w[kWin * kWin];
  static bool init = false;
  if (!init) {
    const int r = kWin / 2;
    double sum = 0.0;
    for (int dy = -r; dy <= r; ++dy)
      for (int dx = -r; dx <= r; ++dx) {
        double v = std::exp(-(dx * dx + dy * dy) / (2.0 * 1.5 * 1.5));
        w[(dy + r) * kWin + (dx + r)] = v;
        sum += v;
      }
    for (double& v : w) v /= sum;
    init = true;
  }
  return w;
}

// Windowed SSIM over valid centres, masked by centre and zero-filled by the
// mask; optionally accumulates grad_scale * d(mean)/d(a) into grad (HWC).
// Returns the mean and writes the sample count.
double ssim_masked(const double* a, const double* b, const double* mask, int w, int h,
                   double* grad, double grad_scale, size_t* n_samples) {
  const int r = kWin / 2;
  const double* wt = ssim_window();
  *n_samples = 0;
  if (w < kWin || h < kWin) return 0.0;
  auto in = [&](int x, int y) { return mask == nullptr || mask[y * w + x] >= 0.5; };
  size_t centers = 0;
  for (int cy = r; cy < h - r; ++cy)
    for (int cx = r; cx < w - r; ++cx)
      if (in(cx, cy)) ++centers;
  if (centers == 0) return 0.0;
  *n_samples = centers * 3;
  const double inv_n = 1.0 / static_cast<double>(*n_samples);
  double total = 0.0;
  for (int cy = r; cy < h - r; ++cy)
    for (int cx = r; cx < w - r; ++cx) {
      if (!in(cx, cy)) continue;
      for (int ch = 0; ch < 3; ++ch) {
        double mx = 0, my = 0, sxx = 0, syy = 0, sxy = 0;
        for (int dy = -r; dy <= r; ++dy)
          for (int dx = -r; dx <= r; ++dx) {
            double wi = wt[(dy + r) * kWin + (dx + r)];
            double m = in(cx + dx, cy + dy) ? 1.0 : 0.0;
            size_t o = (static_cast<size_t>(cy + dy) * w + (cx + dx)) * 3 + ch;
            double xv = a[o] * m, yv = b[o] * m;
            mx += wi * xv;
            my += wi * yv;
            sxx += wi * (xv * xv);
            syy += wi * (yv * yv);
            sxy += wi * (xv * yv);
          }
        double vx = sxx - mx * mx, vy = syy - my * my, cv = sxy - mx * my;
        double a1 = 2.0 * (mx * my) + kC1;
        double b1 = mx * mx + my * my + kC1;
        double a2 = 2.0 * cv + kC2;
        double b2 = vx + vy + kC2;
        double s = (a1 * a2) / (b1 * b2);
        total += s;
        if (grad) {
          double ib = 1.0 / (b1 * b2);
          double coeff = grad_scale * inv_n;
          for (int dy = -r; dy <= r; ++dy)
            for (int dx = -r; dx <= r; ++dx) {
              if (!in(cx + dx, cy + dy)) continue;
              double wi = wt[(dy + r) * kWin + (dx + r)];
              size_t o = (static_cast<size_t>(cy + dy) * w + (cx + dx)) * 3 + ch;
              double xv = a[o], yv = b[o];
              double d = 2.0 * wi * ((my * a2 + (yv - my) * a1) * ib - s * (mx / b1 + (xv - mx) / b2));
              grad[o] += coeff * d;
            }
        }
      }
    }
  return total * inv_n;
}

// masked_loss (loss.hpp:39-73).
double loss_masked(const double* rendered, const double* gt, const double* mask, int w, int h,
                   double lambda, double* dL) {
  size_t np = static_cast<size_t>(w) * h;
  std::fill(dL, dL + 3 * np, 0.0);
  size_t nm = 0;
  for (size_t i = 0; i < np; ++i)
    if (mask[i] >= 0.5) ++nm;
  if (nm == 0) return 0.0;
  const double l1w = (1.0 - lambda) / (static_cast<double>(nm) * 3.0);
  double sum = 0.0;
  for (size_t i = 0; i < np; ++i) {
    if (mask[i] < 0.5) continue;
    for (int c = 0; c < 3; ++c) {
      double d = rendered[3 * i + c] - gt[3 * i + c];
      sum += std::abs(d);
      dL[3 * i + c] = l1w * (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0));
    }
  }
  double loss = (1.0 - lambda) * sum / (static_cast<double>(nm) * 3.0);
  if (lambda > 0.0) {
    size_t ns = 0;
    double mean = ssim_masked(rendered, gt, mask, w, h, dL, -lambda, &ns);
    if (ns > 0) loss += lambda * (1.0 - mean);
  }
  return loss;
}

// ---- forward render (render.hpp:160-205) -----------------------------------
void render_impl(const double* P, int64_t n, const Cam& k, const orc_render_cfg* cfg,
                 double* rgb, double* alpha, int32_t* ncontrib, std::vector<int32_t>* order) {
  const int w = k.w, h = k.h;
  for (size_t i = 0; i < static_cast<size_t>(w) * h; ++i) {
    rgb[3 * i] = cfg->background[0];
    rgb[3 * i + 1] = cfg->background[1];
    rgb[3 * i + 2] = cfg->background[2];
    alpha[i] = 0.0;
    ncontrib[i] = 0;
  }
  std::vector<Splat> s = project_sort(P, n, k, cfg);
  if (order) {
    order->clear();
    for (const Splat& p : s) order->push_back(p.idx);
  }
  if (s.empty()) return;
  Bins b = make_bins(s, w, h, cfg->tile_size);
  const double sig2 = cfg->sigma_cutoff * cfg->sigma_cutoff;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      int t = b.tile_of(x, y);
      double px = x + 0.5, py = y + 0.5, T = 1.0, ar = 0, ag = 0, ab = 0;
      int32_t cnt = 0;
      for (int64_t e = b.start[t]; e < b.start[t + 1]; ++e) {
        const Splat& p = s[static_cast<size_t>(b.pos[static_cast<size_t>(e)])];
        double a, g;
        if (!alpha_at(p, px, py, sig2, cfg->alpha_cutoff, &a, &g)) continue;
        double wgt = a * T;
        ar += p.cr * wgt;
        ag += p.cg * wgt;
        ab += p.cb * wgt;
        ++cnt;
        T *= (1.0 - a);
        if (T < cfg->transmittance_floor) break;
      }
      if (cnt > 0) {
        size_t o = static_cast<size_t>(y) * w + x;
        rgb[3 * o] = ar + cfg->background[0] * T;
        rgb[3 * o + 1] = ag + cfg->background[1] * T;
        rgb[3 * o + 2] = ab + cfg->background[2] * T;
        alpha[o] = 1.0 - T;
        ncontrib[o] = cnt;
      }
    }
}

// ---- backward (backward.hpp:43-332) ----------------------------------------
struct SGrad {  // ScreenGrad, backward.hpp:22-38
  double mx = 0, my = 0;                   // g_mean2d
  double ca = 0, cb = 0, cc = 0, cd = 0;   // g_inv_cov (full 2x2)
  double r = 0, g = 0, b = 0;              // g_color
  double ap = 0;                           // g_alpha_pre
  void add(const SGrad& o) {
    mx = mx + o.mx;
    my = my + o.my;
    ca += o.ca; cb += o.cb; cc += o.cc; cd += o.cd;
    r += o.r; g += o.g; b += o.b;
    ap += o.ap;
  }
};

// d R(q) / d q_k for a unit quaternion (backward.hpp:43-69).
void drot_dq(const double* q, int k, double* m) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  for (int i = 0; i < 9; ++i) m[i] = 0.0;
  switch (k) {
    case 0:
      m[1] = -2 * z; m[2] = 2 * y; m[3] = 2 * z; m[5] = -2 * x; m[6] = -2 * y; m[7] = 2 * x;
      break;
    case 1:
      m[1] = 2 * y; m[2] = 2 * z; m[3] = 2 * y; m[4] = -4 * x; m[5] = -2 * w;
      m[6] = 2 * z; m[7] = 2 * w; m[8] = -4 * x;
      break;
    case 2:
      m[0] = -4 * y; m[1] = 2 * x; m[2] = 2 * w; m[3] = 2 * x; m[5] = 2 * z;
      m[6] = -2 * w; m[7] = 2 * z; m[8] = -4 * y;
      break;
    default:
      m[0] = -4 * z; m[1] = -2 * w; m[2] = 2 * x; m[3] = 2 * w; m[4] = -4 * z; m[5] = 2 * y;
      m[6] = 2 * x; m[7] = 2 * y;
      break;
  }
}

// Screen-space adjoint of rows [r0, r1): per-row subtotals in ascending
// list position (backward.hpp:77-175), folded into `total` in row order by
// the caller (backward.hpp:218-226).
void screen_rows(const std::vector<Splat>& s, const Bins& b, const Cam& k,
                 const orc_render_cfg* cfg, const double* dL, int r0, int r1,
                 std::vector<std::vector<std::pair<int32_t, SGrad>>>* rows) {
  const double sig2 = cfg->sigma_cutoff * cfg->sigma_cutoff;
  std::vector<SGrad> acc(s.size());
  std::vector<uint8_t> seen(s.size(), 0);
  std::vector<int32_t> touched;
  struct Hit {
    int32_t pos;
    double a, T, g;
  };
  std::vector<Hit> stack;
  for (int y = r0; y < r1; ++y) {
    touched.clear();
    for (int x = 0; x < k.w; ++x) {
      int t = b.tile_of(x, y);
      if (b.start[t] == b.start[t + 1]) continue;
      double px = x + 0.5, py = y + 0.5;
      stack.clear();
      double T = 1.0;
      for (int64_t e = b.start[t]; e < b.start[t + 1]; ++e) {
        int32_t pos = b.pos[static_cast<size_t>(e)];
        double a, g;
        if (!alpha_at(s[static_cast<size_t>(pos)], px, py, sig2, cfg->alpha_cutoff, &a, &g))
          continue;
        stack.push_back({pos, a, T, g});
        T *= (1.0 - a);
        if (T < cfg->transmittance_floor) break;
      }
      if (stack.empty()) continue;
      size_t o = (static_cast<size_t>(y) * k.w + x) * 3;
      double wr = dL[o], wg = dL[o + 1], wb = dL[o + 2];
      double br = cfg->background[0] * T, bg = cfg->background[1] * T, bb = cfg->background[2] * T;
      for (size_t j = stack.size(); j-- > 0;) {
        const Hit& c = stack[j];
        const Splat& p = s[static_cast<size_t>(c.pos)];
        SGrad& A = acc[static_cast<size_t>(c.pos)];
        if (!seen[static_cast<size_t>(c.pos)]) {
          seen[static_cast<size_t>(c.pos)] = 1;
          touched.push_back(c.pos);
        }
        double wt = c.a * c.T;
        A.r += wr * wt;
        A.g += wg * wt;
        A.b += wb * wt;
        double inv1m = 1.0 / (1.0 - c.a);
        double ga = wr * (p.cr * c.T - br * inv1m) + wg * (p.cg * c.T - bg * inv1m) +
                    wb * (p.cb * c.T - bb * inv1m);
        if (p.op * c.g <= kAlphaCap) {
          A.ap += ga * c.g;
          double gg = ga * p.op;
          double gq = -0.5 * c.g * gg;
          double dx = px - p.mx, dy = py - p.my;
          double mdx = p.ixx * dx + p.ixy * dy, mdy = p.ixy * dx + p.iyy * dy;
          A.mx = A.mx + mdx * (-2.0 * gq);
          A.my = A.my + mdy * (-2.0 * gq);
          A.ca += gq * dx * dx;
          A.cb += gq * dx * dy;
          A.cc += gq * dy * dx;
          A.cd += gq * dy * dy;
        }
        br = br + p.cr * wt;
        bg = bg + p.cg * wt;
        bb = bb + p.cb * wt;
      }
    }
    std::sort(touched.begin(), touched.end());
    std::vector<std::pair<int32_t, SGrad>> row;
    row.reserve(touched.size());
    for (int32_t pos : touched) {
      row.emplace_back(pos, acc[static_cast<size_t>(pos)]);
      acc[static_cast<size_t>(pos)] = SGrad{};
      seen[static_cast<size_t>(pos)] = 0;
    }
    rows->push_back(std::move(row));
  }
}

void backward_impl(const double* P, int64_t n, const Cam& k, const orc_render_cfg* cfg,
                   const double* dL, double* G, double* dm2, int32_t* touch) {
  std::fill(G, G + 14 * n, 0.0);
  if (dm2) std::fill(dm2, dm2 + 2 * n, 0.0);
  if (touch) std::fill(touch, touch + n, 0);
  std::vector<Splat> s = project_sort(P, n, k, cfg);
  if (s.empty()) return;
  Bins b = make_bins(s, k.w, k.h, cfg->tile_size);
  // Row subtotals are shard-invariant (backward.hpp:194-226), so one band
  // over all rows is the canonical reduction for every shard count.
  std::vector<std::vector<std::pair<int32_t, SGrad>>> rows;
  screen_rows(s, b, k, cfg, dL, 0, k.h, &rows);
  std::vector<SGrad> total(s.size());
  std::vector<uint8_t> any(s.size(), 0);
  for (const auto& row : rows)
    for (const auto& pr : row) {
      total[static_cast<size_t>(pr.first)].add(pr.second);
      any[static_cast<size_t>(pr.first)] = 1;
    }

  const double f = k.f;
  double RT[9];
  mat_T(k.R, RT);
  for (size_t pos = 0; pos < s.size(); ++pos) {
    if (!any[pos]) continue;
    const SGrad& a = total[pos];
    const Splat& p = s[pos];
    const int64_t gi = p.idx;
    const double* g = P + 14 * gi;
    double* out = G + 14 * gi;
    out[11] += a.r;
    out[12] += a.g;
    out[13] += a.b;
    if (dm2) {
      dm2[2 * gi] = dm2[2 * gi] + a.mx;
      dm2[2 * gi + 1] = dm2[2 * gi + 1] + a.my;
    }
    if (touch) touch[gi] = 1;
    out[10] += a.ap * p.op * (1.0 - p.op);

    // dL/dcov2d = -M gM M (backward.hpp:252-261)
    double t1a = p.ixx * a.ca + p.ixy * a.cc, t1b = p.ixx * a.cb + p.ixy * a.cd;
    double t1c = p.ixy * a.ca + p.iyy * a.cc, t1d = p.ixy * a.cb + p.iyy * a.cd;
    double ga = -(t1a * p.ixx + t1b * p.ixy);
    double gb = -(t1a * p.ixy + t1b * p.iyy);
    double gc = -(t1c * p.ixx + t1d * p.ixy);
    double gd = -(t1c * p.ixy + t1d * p.iyy);

    V3 t = to_cam_space(k, {g[0], g[1], g[2]});
    double iz = 1.0 / t.z, iz2 = iz * iz;
    double j00 = f * iz, j02 = -f * t.x * iz2;
    double j11 = -f * iz, j12 = f * t.y * iz2;

    double qn[4], Rq[9], S[9], RS[9], Sc[9];
    quat_unit(g + 6, qn);
    quat_rot(qn[0], qn[1], qn[2], qn[3], Rq);
    double sc[3] = {std::exp(g[3]), std::exp(g[4]), std::exp(g[5])};
    covariance3(g + 3, qn, S);
    mat_mul(k.R, S, RS);
    mat_mul(RS, RT, Sc);

    double J0[3] = {j00, 0.0, j02}, J1[3] = {0.0, j11, j12};
    double gSc[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        gSc[3 * i + j] = J0[i] * (ga * J0[j] + gb * J1[j]) + J1[i] * (gc * J0[j] + gd * J1[j]);

    double sj0[3], sj1[3];
    for (int i = 0; i < 3; ++i) {
      sj0[i] = Sc[3 * i] * J0[0] + Sc[3 * i + 1] * J0[1] + Sc[3 * i + 2] * J0[2];
      sj1[i] = Sc[3 * i] * J1[0] + Sc[3 * i + 1] * J1[1] + Sc[3 * i + 2] * J1[2];
    }
    double gJ0[3], gJ1[3];
    for (int i = 0; i < 3; ++i) {
      gJ0[i] = sj0[i] * (2.0 * ga) + sj1[i] * (gb + gc);
      gJ1[i] = sj0[i] * (gb + gc) + sj1[i] * (2.0 * gd);
    }

    double gtx = a.mx * j00;
    double gty = a.my * j11;
    double gtz = a.mx * (-f * t.x * iz2) + a.my * (f * t.y * iz2);
    gtx += gJ0[2] * (-f * iz2);
    gty += gJ1[2] * (f * iz2);
    gtz += gJ0[0] * (-f * iz2) + gJ0[2] * (2.0 * f * t.x * iz2 * iz) + gJ1[1] * (f * iz2) +
           gJ1[2] * (-2.0 * f * t.y * iz2 * iz);
    // d_mu += R^T g_t (math.hpp:114-118)
    out[0] += k.R[0] * gtx + k.R[3] * gty + k.R[6] * gtz;
    out[1] += k.R[1] * gtx + k.R[4] * gty + k.R[7] * gtz;
    out[2] += k.R[2] * gtx + k.R[5] * gty + k.R[8] * gtz;

    // g_Sigma = R^T gSc R (backward.hpp:296)
    double tmp[9], gS[9];
    mat_mul(RT, gSc, tmp);
    mat_mul(tmp, k.R, gS);

    double M3[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) M3[3 * i + j] = Rq[3 * i + j] * sc[j];
    double gsym[9];
    for (int i = 0; i < 9; ++i) gsym[i] = gS[i] + gS[(i % 3) * 3 + i / 3];
    double gM3[9];
    mat_mul(gsym, M3, gM3);

    for (int c = 0; c < 3; ++c) {
      double gs = 0.0;
      for (int i = 0; i < 3; ++i) gs += gM3[3 * i + c] * Rq[3 * i + c];
      out[3 + c] += gs * sc[c];
    }
    double gR[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) gR[3 * i + j] = gM3[3 * i + j] * sc[j];
    double gqn[4];
    for (int c = 0; c < 4; ++c) {
      double dr[9];
      drot_dq(qn, c, dr);
      double v = 0.0;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) v += gR[3 * i + j] * dr[3 * i + j];
      gqn[c] = v;
    }
    const double* q = g + 6;
    double qnorm = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double d = gqn[0] * qn[0] + gqn[1] * qn[1] + gqn[2] * qn[2] + gqn[3] * qn[3];
    for (int c = 0; c < 4; ++c) out[6 + c] += (gqn[c] - d * qn[c]) / qnorm;
  }
}

// ---- Adam (adam.hpp:55-101) --------------------------------------------------
void adam_impl(double* P, int64_t n, const double* G, double* m, double* v, int64_t* step,
               const double* rates, double b1, double b2, double eps) {
  ++*step;
  double bc1 = 1.0 - std::pow(b1, static_cast<double>(*step));
  double bc2 = 1.0 - std::pow(b2, static_cast<double>(*step));
  static const int group[14] = {0, 0, 0, 1, 1, 1, 2, 2, 2, 2, 3, 4, 4, 4};
  const double lo = std::log(1e-7), hi = std::log(1e3);  // gaussian.hpp:13-14
  for (int64_t i = 0; i < n; ++i) {
    double* p = P + 14 * i;
    for (int s = 0; s < 14; ++s) {
      size_t k = static_cast<size_t>(14 * i + s);
      double gr = G[k];
      m[k] = b1 * m[k] + (1.0 - b1) * gr;
      v[k] = b2 * v[k] + (1.0 - b2) * gr * gr;
      double mh = m[k] / bc1, vh = v[k] / bc2;
      p[s] -= rates[group[s]] * mh / (std::sqrt(vh) + eps);
    }
    double qn[4];
    quat_unit(p + 6, qn);
    for (int c = 0; c < 4; ++c) p[6 + c] = qn[c];
    for (int c = 3; c < 6; ++c) p[c] = std::min(std::max(p[c], lo), hi);
  }
}

// ---- Rng (rng.hpp:8-64) -------------------------------------------------------
struct Rng {
  uint64_t st;
  static uint64_t mix(uint64_t& s) {
    s += 0x9e3779b97f4a7c15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  explicit Rng(uint64_t seed) : st(seed ^ 0x853c49e6748fea9bULL) {
    mix(st);
    mix(st);
  }
  uint64_t u64() { return mix(st); }
  double uni() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
  double normal() {
    double u1 = uni(), u2 = uni();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
  uint64_t below(uint64_t n) { return n > 0 ? u64() % n : 0; }
  template <class T>
  void shuffle(std::vector<T>& v) {
    for (size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[static_cast<size_t>(below(i))]);
  }
};

// ---- densify / prune (trainer.hpp:47-107) ------------------------------------
std::vector<double> densify(const std::vector<double>& P, const std::vector<double>& sg_norm,
                            const std::vector<int32_t>& tcount, const orc_train_cfg* cfg,
                            Rng& rng, std::vector<int32_t>* source) {
  int64_t n = static_cast<int64_t>(P.size() / 14);
  double thr = cfg->split_scale_threshold;
  if (thr <= 0.0) {
    double diag = 0.0;
    if (n > 0) {
      double lo[3] = {P[0], P[1], P[2]}, hi[3] = {P[0], P[1], P[2]};
      for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < 3; ++c) {
          lo[c] = std::min(lo[c], P[14 * i + c]);
          hi[c] = std::max(hi[c], P[14 * i + c]);
        }
      diag = len3({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]});
    }
    thr = 0.02 * diag;
  }
  std::vector<double> out, tail;
  std::vector<int32_t> src, tail_src;
  const double shrink = std::log(0.8);
  for (int64_t i = 0; i < n; ++i) {
    const double* g = &P[static_cast<size_t>(14 * i)];
    if (sigmoid(g[10]) < cfg->prune_opacity) continue;
    double mg = tcount[static_cast<size_t>(i)] > 0 ? sg_norm[static_cast<size_t>(i)] / tcount[static_cast<size_t>(i)] : 0.0;
    if (mg > cfg->densify_grad_threshold) {
      double s[3] = {std::exp(g[3]), std::exp(g[4]), std::exp(g[5])};
      double ms = std::max(s[0], std::max(s[1], s[2]));
      if (ms > thr) {
        double qn[4], R[9];
        quat_unit(g + 6, qn);
        quat_rot(qn[0], qn[1], qn[2], qn[3], R);
        for (int child = 0; child < 2; ++child) {
          double lx = rng.normal() * s[0];
          double ly = rng.normal() * s[1];
          double lz = rng.normal() * s[2];
          double c[14];
          std::memcpy(c, g, sizeof c);
          c[0] = g[0] + (R[0] * lx + R[1] * ly + R[2] * lz);
          c[1] = g[1] + (R[3] * lx + R[4] * ly + R[5] * lz);
          c[2] = g[2] + (R[6] * lx + R[7] * ly + R[8] * lz);
          c[3] = g[3] + shrink;
          c[4] = g[4] + shrink;
          c[5] = g[5] + shrink;
          if (child == 0) {
            out.insert(out.end(), c, c + 14);
            src.push_back(-1);
          } else {
            tail.insert(tail.end(), c, c + 14);
            tail_src.push_back(-1);
          }
        }
      } else {
        out.insert(out.end(), g, g + 14);
        src.push_back(static_cast<int32_t>(i));
        tail.insert(tail.end(), g, g + 14);
        tail_src.push_back(-1);
      }
    } else {
      out.insert(out.end(), g, g + 14);
      src.push_back(static_cast<int32_t>(i));
    }
  }
  out.insert(out.end(), tail.begin(), tail.end());
  src.insert(src.end(), tail_src.begin(), tail_src.end());
  *source = std::move(src);
  return out;
}

// ---- partitioning (partition.hpp:34-126) --------------------------------------
struct Box {
  double lo[3], hi[3];
};
Box bounds_of(const double* pts, int64_t n) {
  Box b{{0, 0, 0}, {0, 0, 0}};
  if (n == 0) return b;
  for (int c = 0; c < 3; ++c) b.lo[c] = b.hi[c] = pts[c];
  for (int64_t i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) {
      double v = pts[3 * i + c];
      b.lo[c] = std::min(b.lo[c], v);
      b.hi[c] = std::max(b.hi[c], v);
    }
  return b;
}
int longest_axis_of(const Box& b) {  // math.hpp:164-170
  double e[3] = {b.hi[0] - b.lo[0], b.hi[1] - b.lo[1], b.hi[2] - b.lo[2]};
  if (e[0] >= e[1] && e[0] >= e[2]) return 0;
  return e[1] >= e[2] ? 1 : 2;
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
const char* orc_impl_name(void) { return "oracle"; }

int orc_prepare(const double* params, int64_t n, const orc_camera* cam, const orc_render_cfg* cfg,
                int64_t* n_out, int32_t* index, double* mean2d, double* inv_cov, double* opacity,
                double* depth, int32_t* rect) {
  return guarded([&] {
    Cam k = make_cam(cam);
    std::vector<Splat> s = project_sort(params, n, k, cfg);
    *n_out = static_cast<int64_t>(s.size());
    for (size_t i = 0; i < s.size(); ++i) {
      index[i] = s[i].idx;
      mean2d[2 * i] = s[i].mx;
      mean2d[2 * i + 1] = s[i].my;
      inv_cov[3 * i] = s[i].ixx;
      inv_cov[3 * i + 1] = s[i].ixy;
      inv_cov[3 * i + 2] = s[i].iyy;
      opacity[i] = s[i].op;
      depth[i] = s[i].depth;
      rect[4 * i] = s[i].x0;
      rect[4 * i + 1] = s[i].x1;
      rect[4 * i + 2] = s[i].y0;
      rect[4 * i + 3] = s[i].y1;
    }
  });
}

int orc_bin(const double* params, int64_t n, const orc_camera* cam, const orc_render_cfg* cfg,
            int32_t* tile_count, int32_t* entries, int64_t capacity, int64_t* n_entries) {
  return guarded([&] {
    Cam k = make_cam(cam);
    std::vector<Splat> s = project_sort(params, n, k, cfg);
    Bins b = make_bins(s, k.w, k.h, cfg->tile_size);
    size_t nt = b.start.size() - 1;
    for (size_t t = 0; t < nt; ++t) tile_count[t] = static_cast<int32_t>(b.start[t + 1] - b.start[t]);
    *n_entries = static_cast<int64_t>(b.pos.size());
    if (*n_entries > capacity) fail(kInvalidArgument, "entry capacity too small");
    for (size_t e = 0; e < b.pos.size(); ++e) entries[e] = s[static_cast<size_t>(b.pos[e])].idx;
  });
}

int orc_render(const double* params, int64_t n, const orc_camera* cam, const orc_render_cfg* cfg,
               double* rgb, double* alpha, int32_t* n_contrib, int32_t* splat_order,
               int64_t* n_order) {
  return guarded([&] {
    validate_cfg(cfg);
    Cam k = make_cam(cam);
    validate_cam(k);
    std::vector<int32_t> order;
    render_impl(params, n, k, cfg, rgb, alpha, n_contrib, &order);
    *n_order = static_cast<int64_t>(order.size());
    if (splat_order) std::copy(order.begin(), order.end(), splat_order);
  });
}

// render_mask (render.hpp:210-233).
int orc_render_mask(const double* points, int64_t n, const orc_camera* cam, double footprint_px,
                    double dilation_px, double* mask) {
  return guarded([&] {
    if (footprint_px < 0.5) fail(kInvalidArgument, "footprint_px must be >= 0.5");
    Cam k = make_cam(cam);
    validate_cam(k);
    std::fill(mask, mask + static_cast<size_t>(k.w) * k.h, 0.0);
    const double rad = footprint_px + dilation_px, rad2 = rad * rad;
    for (int64_t i = 0; i < n; ++i) {
      V3 t = to_cam_space(k, {points[3 * i], points[3 * i + 1], points[3 * i + 2]});
      if (t.z <= k.nearp) continue;
      double u = 0.5 * k.w + k.f * t.x / t.z;
      double v = 0.5 * k.h - k.f * t.y / t.z;
      int x0 = std::max(0, to_int_x86(std::ceil(u - rad - 0.5)));
      int x1 = std::min(k.w - 1, to_int_x86(std::floor(u + rad - 0.5)));
      int y0 = std::max(0, to_int_x86(std::ceil(v - rad - 0.5)));
      int y1 = std::min(k.h - 1, to_int_x86(std::floor(v + rad - 0.5)));
      for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) {
          double dx = x + 0.5 - u, dy = y + 0.5 - v;
          if (dx * dx + dy * dy <= rad2) mask[static_cast<size_t>(y) * k.w + x] = 1.0;
        }
    }
  });
}

int orc_masked_loss(const double* rendered, const double* gt, const double* mask, int32_t width,
                    int32_t height, double lambda, double* loss, double* dL) {
  return guarded([&] { *loss = loss_masked(rendered, gt, mask, width, height, lambda, dL); });
}

int orc_ssim(const double* a, const double* b, int32_t width, int32_t height, double* out) {
  return guarded([&] {
    if (width < kWin || height < kWin) fail(kTooSmall, "images must be at least 11 px per side");
    size_t ns = 0;
    *out = ssim_masked(a, b, nullptr, width, height, nullptr, 1.0, &ns);
  });
}

int orc_psnr(const double* a, const double* b, int64_t count, double* out) {
  return guarded([&] {
    double mse = 0.0;
    for (int64_t i = 0; i < count; ++i) {
      double d = a[i] - b[i];
      mse += d * d;
    }
    mse /= static_cast<double>(count);
    *out = mse <= 0.0 ? 99.0 : std::min(99.0, 10.0 * std::log10(1.0 / mse));
  });
}

int orc_backward(const double* params, int64_t n, int64_t model_iteration,
                 int64_t output_iteration, const orc_camera* cam, const orc_render_cfg* cfg,
                 const double* dL, int32_t shards, double* grads, double* d_mean2d,
                 int32_t* touch) {
  return guarded([&] {
    if (output_iteration != model_iteration)
      fail(kStaleForward, "render output is from a different model iteration");
    if (shards < 1) fail(kInvalidArgument, "shards must be >= 1");
    Cam k = make_cam(cam);
    backward_impl(params, n, k, cfg, dL, grads, d_mean2d, touch);
  });
}

int orc_adam_step(double* params, int64_t n, const double* grads, double* m, double* v,
                  int64_t* step, const double* rates, const double* adam) {
  return guarded([&] { adam_impl(params, n, grads, m, v, step, rates, adam[0], adam[1], adam[2]); });
}

// train_partition_full (trainer.hpp:140-211).
int orc_train(const double* params_in, int64_t n, const orc_camera* cams, const double* gts,
              const double* masks, int32_t n_views, const orc_train_cfg* cfg, int32_t shards,
              double* params_out, int64_t cap_out, int64_t* n_out, double* final_loss,
              double* loss_trace) {
  return guarded([&] {
    if (cfg->lr_mu <= 0 || cfg->lr_scale <= 0 || cfg->lr_rot <= 0 || cfg->lr_opacity <= 0 ||
        cfg->lr_color <= 0)
      fail(kInvalidArgument, "learning rates must be positive");
    if (cfg->loss_lambda < 0.0 || cfg->loss_lambda > 1.0)
      fail(kInvalidArgument, "loss_lambda outside [0, 1]");
    if (cfg->iterations < 0) fail(kInvalidArgument, "iterations must be >= 0");
    if (n_views <= 0) fail(kNoViews, "training requires at least one view");
    if (shards < 1) fail(kInvalidArgument, "shards must be >= 1");
    std::vector<double> P(params_in, params_in + 14 * n);
    *final_loss = 0.0;
    if (cfg->iterations > 0) {
      std::vector<size_t> order(static_cast<size_t>(n_views));
      std::iota(order.begin(), order.end(), size_t{0});
      Rng vr(cfg->seed ^ 0x87aa11d3ULL);
      vr.shuffle(order);
      Rng dr(cfg->seed ^ 0xd3a51f11ULL);
      std::vector<double> m(P.size(), 0.0), v(P.size(), 0.0);
      int64_t step = 0;
      std::vector<double> sg(static_cast<size_t>(n), 0.0);
      std::vector<int32_t> tc(static_cast<size_t>(n), 0);
      const int64_t until =
          static_cast<int64_t>(cfg->densify_stop_fraction * static_cast<double>(cfg->iterations));
      for (int64_t it = 0; it < cfg->iterations; ++it) {
        int32_t vi = static_cast<int32_t>(order[static_cast<size_t>(it) % order.size()]);
        Cam k = make_cam(&cams[vi]);
        validate_cfg(&cfg->render);
        validate_cam(k);
        size_t np = static_cast<size_t>(k.w) * k.h;
        int64_t cur = static_cast<int64_t>(P.size() / 14);
        std::vector<double> rgb(3 * np), al(np), dL(3 * np);
        std::vector<int32_t> nc(np);
        render_impl(P.data(), cur, k, &cfg->render, rgb.data(), al.data(), nc.data(), nullptr);
        double loss = loss_masked(rgb.data(), gts + 3 * np * vi, masks + np * vi, k.w, k.h,
                                  cfg->loss_lambda, dL.data());
        *final_loss = loss;
        std::vector<double> G(P.size()), dm2(2 * static_cast<size_t>(cur));
        std::vector<int32_t> touch(static_cast<size_t>(cur));
        backward_impl(P.data(), cur, k, &cfg->render, dL.data(), G.data(), dm2.data(), touch.data());
        double decay = std::pow(cfg->lr_mu_decay,
                                static_cast<double>(it) / static_cast<double>(cfg->iterations));
        double rates[5] = {cfg->lr_mu * decay, cfg->lr_scale, cfg->lr_rot, cfg->lr_opacity,
                           cfg->lr_color};
        adam_impl(P.data(), cur, G.data(), m.data(), v.data(), &step, rates, cfg->beta1,
                  cfg->beta2, cfg->epsilon);
        // finalize_step_stats + accumulation (gradient.hpp:39-45, trainer.hpp:189-193)
        for (int64_t i = 0; i < cur; ++i) {
          double add = 0.0;
          int32_t t = touch[static_cast<size_t>(i)];
          if (t > 0) {
            add = 0.0 + std::sqrt(dm2[2 * i] * dm2[2 * i] + dm2[2 * i + 1] * dm2[2 * i + 1]);
            t = 1;
          }
          sg[static_cast<size_t>(i)] += add;
          tc[static_cast<size_t>(i)] += t;
        }
        bool now = cfg->densify_interval > 0 && (it + 1) % cfg->densify_interval == 0 &&
                   (it + 1) < until;
        if (now) {
          std::vector<int32_t> src;
          P = densify(P, sg, tc, cfg, dr, &src);
          std::vector<double> nm(src.size() * 14, 0.0), nv(src.size() * 14, 0.0);
          for (size_t j = 0; j < src.size(); ++j) {
            if (src[j] < 0) continue;
            for (int s = 0; s < 14; ++s) {
              nm[14 * j + s] = m[14 * static_cast<size_t>(src[j]) + s];
              nv[14 * j + s] = v[14 * static_cast<size_t>(src[j]) + s];
            }
          }
          m.swap(nm);
          v.swap(nv);
          sg.assign(src.size(), 0.0);
          tc.assign(src.size(), 0);
        }
        if (loss_trace) loss_trace[it] = loss;
      }
    }
    int64_t cur = static_cast<int64_t>(P.size() / 14);
    if (cur > cap_out) fail(kInvalidArgument, "output capacity too small");
    std::copy(P.begin(), P.end(), params_out);
    *n_out = cur;
  });
}

// partition_cloud (partition.hpp:42-104).
int orc_partition(const double* pos, int64_t n, int32_t nparts, double margin, int32_t* axis_out,
                  double* cut_lo, double* cut_hi, double* owned_box, int64_t* owned_count,
                  int64_t* ghost_count, uint32_t* owned_idx, uint32_t* ghost_idx, int64_t cap) {
  return guarded([&] {
    if (n == 0) fail(kEmptyCloud, "cannot partition an empty cloud");
    if (nparts < 1) fail(kInvalidArgument, "partition count must be >= 1");
    if (nparts > n) fail(kInvalidArgument, "more partitions than points");
    if (margin < 0.0) fail(kInvalidArgument, "ghost margin must be >= 0");
    Box box = bounds_of(pos, n);
    int ax = longest_axis_of(box);
    std::vector<uint32_t> ord(static_cast<size_t>(n));
    std::iota(ord.begin(), ord.end(), 0u);
    std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) {
      double va = pos[3 * a + ax], vb = pos[3 * b + ax];
      if (va != vb) return va < vb;
      return a < b;
    });
    std::vector<double> cuts;
    for (int k = 1; k < nparts; ++k) {
      size_t r = static_cast<size_t>(n) * static_cast<size_t>(k) / static_cast<size_t>(nparts);
      cuts.push_back(0.5 * (pos[3 * ord[r - 1] + ax] + pos[3 * ord[r] + ax]));
    }
    const double inf = std::numeric_limits<double>::infinity();
    std::vector<double> lo(static_cast<size_t>(nparts)), hi(static_cast<size_t>(nparts));
    for (int k = 0; k < nparts; ++k) {
      cut_lo[k] = k == 0 ? -inf : cuts[static_cast<size_t>(k - 1)];
      cut_hi[k] = k == nparts - 1 ? inf : cuts[static_cast<size_t>(k)];
      double* b = owned_box + 6 * k;
      for (int c = 0; c < 3; ++c) {
        b[c] = box.lo[c];
        b[3 + c] = box.hi[c];
      }
      if (k > 0) b[ax] = cuts[static_cast<size_t>(k - 1)];
      if (k < nparts - 1) b[3 + ax] = cuts[static_cast<size_t>(k)];
      lo[static_cast<size_t>(k)] = b[ax];
      hi[static_cast<size_t>(k)] = b[3 + ax];
    }
    *axis_out = ax;
    std::vector<std::vector<uint32_t>> own(static_cast<size_t>(nparts)), gh(static_cast<size_t>(nparts));
    for (int64_t i = 0; i < n; ++i) {
      double v = pos[3 * i + ax];
      for (int k = 0; k < nparts; ++k) {
        if (v >= cut_lo[k] && v < cut_hi[k]) {
          own[static_cast<size_t>(k)].push_back(static_cast<uint32_t>(i));
        } else {
          double l = lo[static_cast<size_t>(k)], h = hi[static_cast<size_t>(k)];
          double d = v < l ? l - v : (v > h ? v - h : 0.0);
          if (d <= margin) gh[static_cast<size_t>(k)].push_back(static_cast<uint32_t>(i));
        }
      }
    }
    int64_t oi = 0, gi = 0;
    for (int k = 0; k < nparts; ++k) {
      owned_count[k] = static_cast<int64_t>(own[static_cast<size_t>(k)].size());
      ghost_count[k] = static_cast<int64_t>(gh[static_cast<size_t>(k)].size());
      for (uint32_t x : own[static_cast<size_t>(k)]) {
        if (oi < cap) owned_idx[oi] = x;
        ++oi;
      }
      for (uint32_t x : gh[static_cast<size_t>(k)]) {
        if (gi < cap) ghost_idx[gi] = x;
        ++gi;
      }
    }
    if (oi > cap || gi > cap) fail(kInvalidArgument, "index capacity too small");
  });
}

// merge_models (partition.hpp:109-126): owns() on the final mu.
int orc_merge(const double* params, const int64_t* counts, int32_t nparts, int32_t axis,
              const double* cut_lo, const double* cut_hi, uint8_t* keep, int64_t* n_kept) {
  return guarded([&] {
    int64_t off = 0, kept = 0;
    for (int32_t k = 0; k < nparts; ++k)
      for (int64_t i = 0; i < counts[k]; ++i, ++off) {
        double v = params[14 * off + axis];
        bool o = v >= cut_lo[k] && v < cut_hi[k];
        keep[off] = o ? 1 : 0;
        kept += o;
      }
    *n_kept = kept;
  });
}

// build_orbital_cameras (camera.hpp:75-107).
int orc_orbital_cameras(const double* center, double radius, int32_t n_az, int32_t n_el,
                        int32_t resolution, double fov_y, double max_el, orc_camera* out) {
  return guarded([&] {
    if (n_az < 1 || n_el < 1) fail(kInvalidRig, "azimuth/elevation counts must be >= 1");
    if (!(radius > 0.0)) fail(kInvalidRig, "rig radius must be positive");
    int idx = 0;
    for (int ie = 0; ie < n_el; ++ie) {
      double phi = 0.0;
      if (n_el > 1) phi = -max_el + 2.0 * max_el * ie / (n_el - 1);
      for (int ia = 0; ia < n_az; ++ia) {
        double theta = 2.0 * M_PI * ia / n_az;
        orc_camera& c = out[idx++];
        double dir[3] = {std::cos(phi) * std::cos(theta), std::sin(phi),
                         std::cos(phi) * std::sin(theta)};
        for (int k = 0; k < 3; ++k) {
          c.position[k] = center[k] + dir[k] * radius;
          c.target[k] = center[k];
        }
        c.up[0] = 0; c.up[1] = 1; c.up[2] = 0;
        c.fov_y = fov_y;
        c.width = resolution;
        c.height = resolution;
        c.near_plane = 0.05 * radius;
        c.far_plane = 10.0 * radius;
        validate_cam(make_cam(&c));
      }
    }
  });
}

// split_rig (camera.hpp:116-130).
int orc_split_rig(int64_t n_views, double test_fraction, uint64_t seed, int32_t* train,
                  int64_t* n_train, int32_t* test, int64_t* n_test) {
  return guarded([&] {
    std::vector<int32_t> idx(static_cast<size_t>(n_views));
    std::iota(idx.begin(), idx.end(), 0);
    Rng r(seed ^ 0x5e1170f5ULL);
    r.shuffle(idx);
    int64_t nt = 0;
    if (test_fraction > 0.0 && n_views > 1) {
      nt = std::llround(test_fraction * static_cast<double>(n_views));
      nt = std::min<int64_t>(std::max<int64_t>(nt, 1), n_views - 1);
    }
    *n_train = n_views - nt;
    *n_test = nt;
    for (int64_t i = 0; i < n_views - nt; ++i) train[i] = idx[static_cast<size_t>(i)];
    for (int64_t i = 0; i < nt; ++i) test[i] = idx[static_cast<size_t>(n_views - nt + i)];
  });
}

// knn_mean_distances (seed.hpp:16-35), brute force.
int orc_knn_mean(const double* p, int64_t n, int32_t k, double* out) {
  return guarded([&] {
    std::vector<double> d;
    for (int64_t i = 0; i < n; ++i) {
      d.clear();
      for (int64_t j = 0; j < n; ++j) {
        if (j == i) continue;
        d.push_back(len3({p[3 * i] - p[3 * j], p[3 * i + 1] - p[3 * j + 1], p[3 * i + 2] - p[3 * j + 2]}));
      }
      int kk = std::min<int>(k, static_cast<int>(d.size()));
      out[i] = 0.0;
      if (kk <= 0) continue;
      std::partial_sort(d.begin(), d.begin() + kk, d.end());
      double s = 0.0;
      for (int m = 0; m < kk; ++m) s += d[static_cast<size_t>(m)];
      out[i] = s / kk;
    }
  });
}

// median_nn_spacing (seed.hpp:39-45).
int orc_median_nn(const double* p, int64_t n, double* out) {
  if (n == 0) return guarded([&] { fail(kEmptyCloud, "empty point cloud"); });
  if (n == 1) {
    *out = 1.0;
    return 0;
  }
  std::vector<double> nn(static_cast<size_t>(n));
  int rc = orc_knn_mean(p, n, 1, nn.data());
  if (rc) return rc;
  std::nth_element(nn.begin(), nn.begin() + n / 2, nn.end());
  *out = nn[static_cast<size_t>(n / 2)];
  return 0;
}

// seed_gaussians(Knn) (seed.hpp:49-74).
int orc_seed_knn(const double* p, const double* colors, int64_t n, int32_t k, double* params) {
  if (n == 0) return guarded([&] { fail(kEmptyCloud, "cannot seed from an empty cloud"); });
  std::vector<double> sc;
  if (n > 1) {
    sc.resize(static_cast<size_t>(n));
    int rc = orc_knn_mean(p, n, k, sc.data());
    if (rc) return rc;
  }
  const double op = std::log(0.1 / (1.0 - 0.1));
  for (int64_t i = 0; i < n; ++i) {
    double s = sc.empty() ? 0.01 : std::max(sc[static_cast<size_t>(i)], 1e-7);
    double ls = std::log(s);
    double* g = params + 14 * i;
    g[0] = p[3 * i]; g[1] = p[3 * i + 1]; g[2] = p[3 * i + 2];
    g[3] = g[4] = g[5] = ls;
    g[6] = 1.0; g[7] = g[8] = g[9] = 0.0;
    g[10] = op;
    g[11] = colors[3 * i]; g[12] = colors[3 * i + 1]; g[13] = colors[3 * i + 2];
  }
  return 0;
}

// ground_truth_model (seed.hpp:78-94).
int orc_gt_model(const double* p, const double* colors, int64_t n, double scale, double opacity,
                 double* params) {
  return guarded([&] {
    if (n == 0) fail(kEmptyCloud, "cannot build ground truth from nothing");
    double ls = std::log(std::max(scale, 1e-7));
    double lo = std::log(opacity / (1.0 - opacity));
    for (int64_t i = 0; i < n; ++i) {
      double* g = params + 14 * i;
      g[0] = p[3 * i]; g[1] = p[3 * i + 1]; g[2] = p[3 * i + 2];
      g[3] = g[4] = g[5] = ls;
      g[6] = 1.0; g[7] = g[8] = g[9] = 0.0;
      g[10] = lo;
      g[11] = colors[3 * i]; g[12] = colors[3 * i + 1]; g[13] = colors[3 * i + 2];
    }
  });
}

int orc_rng_uniform(uint64_t seed, int64_t count, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = r.uni();
  return 0;
}

}  // extern "C"
