// K8 masked L1 + D-SSIM loss and its pixel gradient (sm_100a).
//
// Replaces masked_loss (loss.hpp:39-73) and ssim_core (ssim.hpp:48-121).
// The 11x11 Gaussian window (sigma 1.5, ssim.hpp:17-31) is separable, so the
// windowed statistics are two 11-tap passes through shared memory instead
// of 121-tap loops; the analytic gradient
//   d ssim_c / d x_p = 2 w(p-c) [ P_c + y_p Q_c - x_p R_c ]
// (expanding ssim.hpp:109-113) turns into a second separable correlation
// of the per-centre coefficients P, Q, R. Statistics, coefficients and the
// correlations are fp64 (the variance terms cancel catastrophically in
// fp32); the per-block partial sums are folded in a fixed order, so the
// loss is deterministic.
//
//   k_ssim_stats : per centre -> P, Q, R (zero unless a valid masked centre),
//                  block SSIM partial sums, mask / centre counts
//   k_loss_grad  : per pixel  -> dL (L1 sign term + SSIM correlation), L1 partials
//   k_loss_final : one block  -> loss scalar
#include "dsg_internal.h"
#include "raster.h"

namespace dsg {

namespace {

constexpr int kW = 11, kR = 5;
constexpr int kB = 16;             // output block edge
constexpr int kE = kB + 2 * kR;    // 26: block plus apron
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;  // ssim.hpp:12-13

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed shuffle tree + fixed warp order).
__device__ double block_sum_d(double v, double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum_d(v);
  __syncthreads();
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sm[w];
  return t;
}

struct LossArgs {
  const float* x;      // rendered, planar [3][npix]
  const float* y;      // ground truth, planar [3][npix]
  const uint8_t* m;    // mask [npix]
  int w, h;
  int64_t npix;
  double lambda;
  double* pqr;         // [3 ch][3][npix]
  double* parts;       // [blocks] ssim partials, then [blocks] l1 partials
  uint32_t* counts;    // [0] masked pixels, [1] valid masked centres
  float* dL;           // planar [3][npix]
  double* loss_out;
  int nblocks;
  // 1-D factor of the SSIM window (outer product sums to 1, ssim.hpp:17-31);
  // a kernel parameter, so every device and context sees it with the launch
  double win[kW];
};

__global__ void __launch_bounds__(kB* kB) k_ssim_stats(LossArgs a) {
  DSG_PDL_ENTRY();
  __shared__ double xs[kE][kE], ys[kE][kE];
  __shared__ double hs[5][kE][kB];
  __shared__ double red[32];
  const int bx = blockIdx.x * kB, by = blockIdx.y * kB;
  const int tx = threadIdx.x % kB, ty = threadIdx.x / kB;
  const int cx = bx + tx, cy = by + ty;
  const bool in_img = cx < a.w && cy < a.h;
  const bool centre_in = in_img && a.m[(int64_t)cy * a.w + cx] != 0;
  const bool valid = centre_in && cx >= kR && cx < a.w - kR && cy >= kR && cy < a.h - kR;
  // counts (integer atomics: order independent)
  uint32_t nm = __syncthreads_count(centre_in);
  uint32_t nc = __syncthreads_count(valid);
  if (threadIdx.x == 0) {
    if (nm) atomicAdd(&a.counts[0], nm);
    if (nc) atomicAdd(&a.counts[1], nc);
  }
  double ssum = 0.0;
  if (nc == 0) {  // no valid masked centre in this block: P = Q = R = 0
    if (in_img) {
      const int64_t o = (int64_t)cy * a.w + cx;
#pragma unroll
      for (int k = 0; k < 9; ++k) a.pqr[k * a.npix + o] = 0.0;
    }
    if (threadIdx.x == 0) a.parts[blockIdx.y * gridDim.x + blockIdx.x] = 0.0;
    return;
  }
  for (int ch = 0; ch < 3; ++ch) {
    const float* X = a.x + ch * a.npix;
    const float* Y = a.y + ch * a.npix;
    for (int t = threadIdx.x; t < kE * kE; t += kB * kB) {
      int r = t / kE, c = t % kE;
      int gx = bx - kR + c, gy = by - kR + r;
      double xv = 0.0, yv = 0.0;
      if (gx >= 0 && gx < a.w && gy >= 0 && gy < a.h) {
        int64_t o = (int64_t)gy * a.w + gx;
        if (a.m[o]) {
          xv = X[o];
          yv = Y[o];
        }
      }
      xs[r][c] = xv;
      ys[r][c] = yv;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < kE * kB; t += kB * kB) {
      int r = t / kB, c = t % kB;
      double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
#pragma unroll
      for (int k = 0; k < kW; ++k) {
        double wk = a.win[k], xv = xs[r][c + k], yv = ys[r][c + k];
        s0 += wk * xv;
        s1 += wk * yv;
        s2 += wk * (xv * xv);
        s3 += wk * (yv * yv);
        s4 += wk * (xv * yv);
      }
      hs[0][r][c] = s0; hs[1][r][c] = s1; hs[2][r][c] = s2; hs[3][r][c] = s3; hs[4][r][c] = s4;
    }
    __syncthreads();
    double P = 0, Q = 0, R = 0;
    if (valid) {
      double mx = 0, my = 0, sxx = 0, syy = 0, sxy = 0;
#pragma unroll
      for (int k = 0; k < kW; ++k) {
        double wk = a.win[k];
        mx += wk * hs[0][ty + k][tx];
        my += wk * hs[1][ty + k][tx];
        sxx += wk * hs[2][ty + k][tx];
        syy += wk * hs[3][ty + k][tx];
        sxy += wk * hs[4][ty + k][tx];
      }
      double vx = sxx - mx * mx, vy = syy - my * my, cv = sxy - mx * my;
      double a1 = 2.0 * (mx * my) + kC1, b1 = mx * mx + my * my + kC1;
      double a2 = 2.0 * cv + kC2, b2 = vx + vy + kC2;
      double s = (a1 * a2) / (b1 * b2);
      ssum += s;
      double ib = 1.0 / (b1 * b2);
      P = my * (a2 - a1) * ib - s * mx / b1 + s * mx / b2;
      Q = a1 * ib;
      R = s / b2;
    }
    if (in_img) {
      int64_t o = (int64_t)cy * a.w + cx;
      a.pqr[(ch * 3 + 0) * a.npix + o] = P;
      a.pqr[(ch * 3 + 1) * a.npix + o] = Q;
      a.pqr[(ch * 3 + 2) * a.npix + o] = R;
    }
    __syncthreads();
  }
  double t = block_sum_d(ssum, red);
  if (threadIdx.x == 0) a.parts[blockIdx.y * gridDim.x + blockIdx.x] = t;
}

__global__ void __launch_bounds__(kB* kB) k_loss_grad(LossArgs a) {
  DSG_PDL_ENTRY();
  __shared__ double ps[3][kE][kE];
  __shared__ double hs[3][kE][kB];
  __shared__ double red[32];
  const int bx = blockIdx.x * kB, by = blockIdx.y * kB;
  const int tx = threadIdx.x % kB, ty = threadIdx.x / kB;
  const int px = bx + tx, py = by + ty;
  const bool in_img = px < a.w && py < a.h;
  const int64_t o = (int64_t)py * a.w + px;
  const bool min = in_img && a.m[o] != 0;
  const uint32_t n_masked = a.counts[0], n_centres = a.counts[1];
  // dL is zero off the mask: a block without a masked pixel has nothing to do
  if (__syncthreads_count(min) == 0) {
    if (in_img) {
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) a.dL[ch * a.npix + o] = 0.f;
    }
    if (threadIdx.x == 0) a.parts[a.nblocks + blockIdx.y * gridDim.x + blockIdx.x] = 0.0;
    return;
  }
  const bool use_ssim = a.lambda > 0.0 && n_centres > 0;
  const double l1w = n_masked ? (1.0 - a.lambda) / ((double)n_masked * 3.0) : 0.0;
  const double coeff = use_ssim ? -a.lambda / ((double)n_centres * 3.0) : 0.0;
  double l1 = 0.0;
  for (int ch = 0; ch < 3; ++ch) {
    double corr[3] = {0, 0, 0};
    if (use_ssim) {
      for (int t = threadIdx.x; t < kE * kE; t += kB * kB) {
        int r = t / kE, c = t % kE;
        int gx = bx - kR + c, gy = by - kR + r;
        bool ok = gx >= 0 && gx < a.w && gy >= 0 && gy < a.h;
        int64_t g = (int64_t)gy * a.w + gx;
#pragma unroll
        for (int k = 0; k < 3; ++k) ps[k][r][c] = ok ? a.pqr[(ch * 3 + k) * a.npix + g] : 0.0;
      }
      __syncthreads();
      for (int t = threadIdx.x; t < kE * kB; t += kB * kB) {
        int r = t / kB, c = t % kB;
        double s0 = 0, s1 = 0, s2 = 0;
#pragma unroll
        for (int k = 0; k < kW; ++k) {
          double wk = a.win[k];
          s0 += wk * ps[0][r][c + k];
          s1 += wk * ps[1][r][c + k];
          s2 += wk * ps[2][r][c + k];
        }
        hs[0][r][c] = s0; hs[1][r][c] = s1; hs[2][r][c] = s2;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kW; ++k) {
        double wk = a.win[k];
        corr[0] += wk * hs[0][ty + k][tx];
        corr[1] += wk * hs[1][ty + k][tx];
        corr[2] += wk * hs[2][ty + k][tx];
      }
      __syncthreads();
    }
    if (in_img) {
      double g = 0.0;
      if (min) {
        double xv = a.x[ch * a.npix + o], yv = a.y[ch * a.npix + o];
        double diff = xv - yv;
        l1 += fabs(diff);
        g = l1w * (diff > 0.0 ? 1.0 : (diff < 0.0 ? -1.0 : 0.0));
        if (use_ssim) g += coeff * 2.0 * (corr[0] + yv * corr[1] - xv * corr[2]);
      }
      a.dL[ch * a.npix + o] = (float)g;
    }
  }
  double t = block_sum_d(l1, red);
  if (threadIdx.x == 0) a.parts[a.nblocks + blockIdx.y * gridDim.x + blockIdx.x] = t;
}

__global__ void __launch_bounds__(256) k_loss_final(LossArgs a) {
  DSG_PDL_ENTRY();
  __shared__ double red[32];
  double s = 0.0, l = 0.0;
  // fixed per-thread strided order, then fixed tree: deterministic
  for (int i = threadIdx.x; i < a.nblocks; i += blockDim.x) {
    s += a.parts[i];
    l += a.parts[a.nblocks + i];
  }
  double ss = block_sum_d(s, red);
  __syncthreads();
  double ll = block_sum_d(l, red);
  if (threadIdx.x == 0) {
    const uint32_t nm = a.counts[0], nc = a.counts[1];
    double loss = 0.0;
    if (nm) {
      loss = (1.0 - a.lambda) * ll / ((double)nm * 3.0);
      if (a.lambda > 0.0 && nc) loss += a.lambda * (1.0 - ss / ((double)nc * 3.0));
    }
    a.loss_out[0] = loss;
  }
}

// Squared error per block (psnr, metrics.hpp:20-30), fp64, deterministic.
__global__ void __launch_bounds__(kB* kB) k_sq_err(LossArgs a) {
  __shared__ double red[32];
  const int cx = blockIdx.x * kB + threadIdx.x % kB, cy = blockIdx.y * kB + threadIdx.x / kB;
  double e = 0.0;
  if (cx < a.w && cy < a.h) {
    const int64_t o = (int64_t)cy * a.w + cx;
    for (int ch = 0; ch < 3; ++ch) {
      const double d = (double)a.x[ch * a.npix + o] - (double)a.y[ch * a.npix + o];
      e += d * d;
    }
  }
  const double t = block_sum_d(e, red);
  if (threadIdx.x == 0) a.parts[a.nblocks + blockIdx.y * gridDim.x + blockIdx.x] = t;
}

// out[0] = psnr (kPsnrCap 99 when identical), out[1] = mean windowed SSIM
// over the valid centres (metrics.hpp:20-38, ssim.hpp:48-121)
__global__ void __launch_bounds__(256) k_metric_final(LossArgs a) {
  __shared__ double red[32];
  double s = 0.0, l = 0.0;
  for (int i = threadIdx.x; i < a.nblocks; i += blockDim.x) {
    s += a.parts[i];
    l += a.parts[a.nblocks + i];
  }
  const double ss = block_sum_d(s, red);
  __syncthreads();
  const double se = block_sum_d(l, red);
  if (threadIdx.x == 0) {
    const double mse = se / (double)(3 * a.npix);
    a.loss_out[0] = mse <= 0.0 ? 99.0 : fmin(99.0, 10.0 * log10(1.0 / mse));
    const uint32_t nc = a.counts[1];
    a.loss_out[1] = nc ? ss / ((double)nc * 3.0) : 0.0;
  }
}

// gaussian_window (ssim.hpp:17-31) factored: g_k / sum(g), sigma 1.5
void fill_window(double* g) {
  double sum = 0.0;
  for (int k = 0; k < kW; ++k) {
    int d = k - kR;
    g[k] = exp(-(double)(d * d) / (2.0 * 1.5 * 1.5));
    sum += g[k];
  }
  for (int k = 0; k < kW; ++k) g[k] /= sum;
}

}  // namespace

void masked_loss_dev(Frame& f, const float* gt, const uint8_t* mask, int width, int height,
                     double lambda, cudaStream_t st, double* out) {
  const int64_t npix = (int64_t)width * height;
  dim3 grid((width + kB - 1) / kB, (height + kB - 1) / kB);
  const int nblocks = grid.x * grid.y;
  f.dL.ensure(3 * npix);
  f.ssim_pqr.ensure(9 * npix);
  f.loss_parts.ensure(2 * nblocks);
  f.loss_counts.ensure(2);
  f.loss_out.ensure(1);
  DSG_CUDA_CHECK(cudaMemsetAsync(f.loss_counts.get(), 0, 2 * sizeof(uint32_t), st));
  LossArgs a;
  a.x = f.rgb.get();
  a.y = gt;
  a.m = mask;
  a.w = width;
  a.h = height;
  a.npix = npix;
  a.lambda = lambda;
  a.pqr = f.ssim_pqr.get();
  a.parts = f.loss_parts.get();
  a.counts = f.loss_counts.get();
  a.dL = f.dL.get();
  a.loss_out = out ? out : f.loss_out.get();
  a.nblocks = nblocks;
  fill_window(a.win);
  pdl_launch(k_ssim_stats, grid, kB * kB, 0, st, a);
  count_launch();
  pdl_launch(k_loss_grad, grid, kB * kB, 0, st, a);
  count_launch();
  pdl_launch(k_loss_final, 1, 256, 0, st, a);
  count_launch();
  DSG_CUDA_CHECK(cudaGetLastError());
}

// psnr and ssim (metrics.hpp:20-38) of two planar fp32 RGB images on the
// device; out (device) receives {psnr, ssim}.
void image_metrics_dev(Frame& f, const float* x, const float* y, int width, int height,
                       cudaStream_t st, double* out) {
  const int64_t npix = (int64_t)width * height;
  dim3 grid((width + kB - 1) / kB, (height + kB - 1) / kB);
  const int nblocks = grid.x * grid.y;
  f.ssim_pqr.ensure(9 * npix);
  f.loss_parts.ensure(2 * nblocks);
  f.loss_counts.ensure(2);
  uint8_t* ones = f.ones_mask.ensure(npix);
  DSG_CUDA_CHECK(cudaMemsetAsync(ones, 1, npix, st));
  DSG_CUDA_CHECK(cudaMemsetAsync(f.loss_counts.get(), 0, 2 * sizeof(uint32_t), st));
  LossArgs a{};
  a.x = x;
  a.y = y;
  a.m = ones;
  a.w = width;
  a.h = height;
  a.npix = npix;
  a.pqr = f.ssim_pqr.get();
  a.parts = f.loss_parts.get();
  a.counts = f.loss_counts.get();
  a.loss_out = out;
  a.nblocks = nblocks;
  fill_window(a.win);
  pdl_launch(k_ssim_stats, grid, kB * kB, 0, st, a);
  k_sq_err<<<grid, kB * kB, 0, st>>>(a);
  k_metric_final<<<1, 256, 0, st>>>(a);
  count_launch(3);
  DSG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace dsg
