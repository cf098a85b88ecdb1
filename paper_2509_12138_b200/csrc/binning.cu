// K1 preprocess, depth-sort fix-up, K2 duplicate, K4 tile ranges (sm_100a).
//
// K1 replaces try_project (projection.hpp:24-57) and the cull/rect part of
// prepare_splats (render.hpp:62-97). Every integer- or order-producing value
// (camera-space depth, mean2d, cov2d, pixel rect, culling) is computed in
// exact fp64 without FMA contraction, so rects, tile counts and the sorted
// key lists match the x86-64 reference bit-for-bit; the blend payload is
// stored as fp32 (mean2d as a hi/lo pair so pixel offsets stay exact).
//
// Ordering: visible splats are sorted by a 32-bit key, the fp64 depth
// quantised over the visible depth range (monotone in the fp64 depth); the
// compaction is index-ordered and the sort stable, so only runs of equal keys
// with out-of-order neighbours need work: short ones are insertion-sorted,
// long ones radix-sorted by fp64 depth bits, and past kLongCap long runs the
// whole visible set is sorted by (fp64 depth bits, index) — the reference
// comparator (render.hpp:98-101). The duplicates are then stably sorted by
// tile id, so every tile list is in reference compositing order.
#include <atomic>
#include <cstdlib>

#include "dsg_internal.h"
#include "raster.h"
#include "scan_util.cuh"

namespace dsg {

namespace {

#ifndef DSG_PRE_QEFF32
#define DSG_PRE_QEFF32 1
#endif
#ifndef DSG_PRE_MINB
#define DSG_PRE_MINB 5  // 5 CTAs/SM (48 regs): measured 0.27 vs 0.30 ms
#endif
__global__ void __launch_bounds__(256, DSG_PRE_MINB) k_preprocess(PreprocessArgs a) {
  DSG_PDL_ENTRY();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  bool vis = false;
  double dep = 0.0;
  if (i < a.n) {
    double p[kParams];
#pragma unroll
    for (int k = 0; k < kParams; ++k) p[k] = (double)a.params[(int64_t)k * a.pitch + i];
    Proj64 pr;
    uint32_t count = 0;
    if (project64(p, a.cam, pr)) {
      double rx = dm(a.rd.sigma_cutoff, sqrt(pr.cxx));
      double ry = dm(a.rd.sigma_cutoff, sqrt(pr.cyy));
      int x0 = max(to_int_x86(ceil(ds(ds(pr.mx, rx), 0.5))), 0);
      int x1 = min(to_int_x86(floor(ds(da(pr.mx, rx), 0.5))), a.cam.width - 1);
      int y0 = max(to_int_x86(ceil(ds(ds(pr.my, ry), 0.5))), 0);
      int y1 = min(to_int_x86(floor(ds(da(pr.my, ry), 0.5))), a.cam.height - 1);
      double det = ds(dm(pr.cxx, pr.cyy), dm(pr.cxy, pr.cxy));
      // tile-parallel global render: only splats reaching this rank's band
      const int bty0 = max(y0 / kTile, a.cam.band_ty0), bty1 = min(y1 / kTile, a.cam.band_ty1 - 1);
      if (x0 <= x1 && y0 <= y1 && det > 0.0 && bty0 <= bty1) {
        double ixx = dd(pr.cyy, det), ixy = dd(-pr.cxy, det), iyy = dd(pr.cxx, det);
        double op = sigmoid64(p[10]);
        // conditioning of the conic: bounds the fp32 rounding of q (guard band)
        double tr = ixx + iyy, df = ixx - iyy;
        double lmax = 0.5 * (tr + sqrt(df * df + 4.0 * ixy * ixy));
        double lmin = (1.0 / det) / lmax;
        double kappa = (fabs(ixx) + fabs(iyy) + 2.0 * fabs(ixy)) / lmin;
        float mxh = (float)pr.mx, myh = (float)pr.my;
        float4* r = a.rec + 3 * i;
        r[0] = make_float4(mxh, myh, (float)(pr.mx - (double)mxh), (float)(pr.my - (double)myh));
        r[1] = make_float4((float)ixx, (float)ixy, (float)iyy, (float)op);
        r[2] = make_float4((float)p[11], (float)p[12], (float)p[13], (float)kappa);
        int tx0 = x0 / kTile, tx1 = x1 / kTile;
        a.trect[i] = make_int4(x0, y0, x1, y1);  // pixel rect; tile rect = rect / kTile
        // Effective rect for the blend's sub-tile masks: alpha >= cutoff needs
        // o*exp(-q/2) >= c, i.e. q <= 2 ln(o/c), so only pixels with
        // |d| <= sqrt(q_eff * cov) can composite (widened by one pixel).
#if DSG_PRE_QEFF32
        // only bounds depend on q_eff (masks and effective rects are
        // conservative), so fp32 log with a 1e-5 pad — two orders above its
        // error — replaces the fp64 log
        const double q_eff = fmin(
            a.rd.sigma_sq,
            (double)(2.f * logf((float)op / a.rd.alpha_cutoff_f)) * (1.0 + 1e-6) + 1e-5);
        {  // sub-tile mask constants (see subtile_mask): ixy/ixx, 1/ixx, q0, qcut
          const double inv = 1.0 / ixx, rr = ixy * inv;
          a.mrow[i] = make_float4((float)rr, (float)inv, (float)(iyy - ixy * rr), (float)q_eff);
        }
#else
        const double q_eff = fmin(a.rd.sigma_sq, 2.0 * log(op / a.rd.alpha_cutoff));
        {  // sub-tile mask constants (see subtile_mask): ixy/ixx, 1/ixx, q0, qcut
          const double inv = 1.0 / ixx, rr = ixy * inv;
          a.mrow[i] = make_float4((float)rr, (float)inv, (float)(iyy - ixy * rr),
                                  (float)(q_eff + 1e-9 * fabs(q_eff) + 1e-12));
        }
#endif
        if (q_eff < 0.0) {
          a.erect[i] = make_int4(1, 1, 0, 0);  // never composites anywhere
        } else {
          const double ex = sqrt(q_eff * pr.cxx), ey = sqrt(q_eff * pr.cyy);
          a.erect[i] = make_int4((int)ceil(pr.mx - ex - 0.5) - 1, (int)ceil(pr.my - ey - 0.5) - 1,
                                 (int)floor(pr.mx + ex - 0.5) + 1, (int)floor(pr.my + ey - 0.5) + 1);
        }
        count = (uint32_t)((tx1 - tx0 + 1) * (bty1 - bty0 + 1));
        a.depth[i] = pr.depth;
        double2* ex = a.exact + 3 * i;
        ex[0] = make_double2(pr.mx, pr.my);
        ex[1] = make_double2(ixx, ixy);
        ex[2] = make_double2(iyy, op);
        dep = pr.depth;
        vis = true;
      }
    }
    a.tcount[i] = count;
  }
  // fp64 depth range of the visible set (positive doubles order like their
  // bits): the depth keys quantise [dmin, dmax] to 32 bits (k_vis_compact)
  unsigned long long dmin = vis ? (unsigned long long)__double_as_longlong(dep) : ~0ull;
  unsigned long long dmax = vis ? (unsigned long long)__double_as_longlong(dep) : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dmin = min(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
    dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  }
  // one pair of atomics per block, and only when it can move the bound
  // (same-address atomics from every warp serialise in L2)
  __shared__ unsigned long long smin[8], smax[8];
  const int warp = threadIdx.x >> 5;
  if (lane == 0) {
    smin[warp] = dmin;
    smax[warp] = dmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      dmin = min(dmin, smin[w]);
      dmax = max(dmax, smax[w]);
    }
    volatile unsigned long long* c = a.drange;
    if (dmin < c[0]) atomicMin(a.drange, dmin);
    if (dmax > c[1]) atomicMax(a.drange + 1, dmax);
  }
}

// Depth key width (radix passes = bits / 8). Runs of equal keys (depths
// within range / 2^bits) are put in (depth, index) order by the fix-up below;
// 24 bits saves a pass at N=1 but makes long near-coincident runs (and their
// radix-sort fallback) far more frequent in sparse partition views.
// Backward partial rows keyed by splat index (1) or by duplicate emission
// position (0); see bin_frame.
#ifndef DSG_ROWS_BY_INDEX
#define DSG_ROWS_BY_INDEX 1
#endif
#ifndef DSG_DEPTH_KEY_BITS
#define DSG_DEPTH_KEY_BITS 32
#endif
constexpr int kDepthKeyBits = DSG_DEPTH_KEY_BITS;

// Order-preserving compaction of the visible set (slot = scan of tcount != 0).
// The key is the fp64 depth quantised over [dmin, dmax] to 32 bits: monotone
// in the fp64 depth, and equal only for depths within range / 2^32, so the
// (depth, index) fix-up below has (almost) nothing to do.
__global__ void k_vis_compact(const uint32_t* __restrict__ tcount, const double* __restrict__ depth,
                              const unsigned long long* __restrict__ drange,
                              const uint32_t* __restrict__ slot, int64_t n,
                              uint32_t* __restrict__ vis_key, uint32_t* __restrict__ vis_idx) {
  DSG_PDL_ENTRY();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || tcount[i] == 0) return;
  const double lo = __longlong_as_double((long long)drange[0]);
  const double hi = __longlong_as_double((long long)drange[1]);
  const double kmax = (double)((1u << kDepthKeyBits) - 1u);
  const double scale = hi > lo ? kmax / (hi - lo) : 0.0;
  const double q = floor((depth[i] - lo) * scale);
  const uint32_t s = slot[i];
  vis_key[s] = q >= kmax ? (uint32_t)kmax : (uint32_t)q;
  vis_idx[s] = (uint32_t)i;
}

// Runs of equal keys must end in (fp64 depth, index) order, the reference
// comparator (render.hpp:98-101). They arrive index-ordered (index-ordered
// compaction, stable sort), so exact depth ties are already right; only
// depths closer than the key quantum can be out of order. Pass 1 marks, at
// its run start, every run holding an out-of-order neighbour pair (read-only
// walk back); pass 2 insertion-sorts just those runs.
__device__ __forceinline__ bool depth_before(uint32_t u, uint32_t v, const double* depth) {
  const double du = depth[u], dv = depth[v];
  return du < dv || (du == dv && u < v);
}

__global__ void k_depth_mark(const uint32_t* __restrict__ key, const uint32_t* __restrict__ idx,
                             int64_t n, const double* __restrict__ depth,
                             uint32_t* __restrict__ runflag) {
  DSG_PDL_ENTRY();
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s + 1 >= n) return;
  const uint32_t k = key[s];
  if (key[s + 1] != k || depth_before(idx[s], idx[s + 1], depth)) return;
  int64_t b = s;
  while (b > 0 && key[b - 1] == k) --b;
  runflag[b] = 1;
}

constexpr int kFixSerial = 64;  // longer flagged runs get a radix sort (bin_frame)

__global__ void k_depth_fixup(const uint32_t* __restrict__ key, uint32_t* idx, int64_t n,
                              const double* __restrict__ depth,
                              const uint32_t* __restrict__ runflag, uint32_t* long_runs,
                              uint32_t long_cap) {
  DSG_PDL_ENTRY();
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n || !runflag[s]) return;
  const uint32_t k = key[s];
  int64_t e = s + 1;
  while (e < n && key[e] == k) ++e;
  if (e - s > kFixSerial) {  // long run (many near-coincident splats): sorted separately
    const uint32_t slot = atomicAdd(long_runs, 1u);
    if (slot < long_cap) {
      long_runs[1 + 2 * slot] = (uint32_t)s;
      long_runs[2 + 2 * slot] = (uint32_t)(e - s);
    }
    return;
  }
  for (int64_t j = s + 1; j < e; ++j) {
    const uint32_t v = idx[j];
    int64_t m = j - 1;
    while (m >= s && !depth_before(idx[m], v, depth)) {
      idx[m + 1] = idx[m];
      --m;
    }
    idx[m + 1] = v;
  }
}

// Long run [s, s+len): (fp64 depth bits, index) pairs for a stable radix
// sort by depth; the run arrives index-ordered, so ties end index-ordered.
__global__ void k_run_keys(const uint32_t* __restrict__ idx, uint32_t s, uint32_t len,
                           const double* __restrict__ depth, unsigned long long* keys,
                           uint32_t* vals) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= len) return;
  const uint32_t v = idx[s + j];
  keys[j] = (unsigned long long)__double_as_longlong(depth[v]);
  vals[j] = v;
}

__global__ void k_gather_counts(const uint32_t* __restrict__ vis_idx, int64_t nv,
                                const uint32_t* __restrict__ tcount, uint32_t* out) {
  DSG_PDL_ENTRY();
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nv) out[s] = tcount[vis_idx[s]];
}

// Sub-tile mask of one (splat, tile): bit (sy*2 + sx) for every 8x4 sub-tile
// holding a pixel centre the splat can composite at. Compositing needs
// q <= sigma^2 and o*exp(-q/2) >= alpha_cutoff (render.hpp:140-154), i.e.
// q <= q_eff = min(sigma^2, 2 ln(o/alpha_cutoff)); the blend's fp32 path
// agrees with fp64 on every such decision (guard band), so the composited
// set is the fp64 one. With q = ixx (dx - dx*)^2 + q0 dy^2, each pixel row's
// q <= qcut set is the x interval centred at dx* = -ixy dy / ixx with
// half-width sqrt((qcut - q0 dy^2) / ixx). Per splat the constants are
// formed by K1 (qcut = q_eff padded by 1e-5 over its fp32 log); per row they are evaluated
// in fp32 (mean2d as hi/lo pairs, so dy is exact to ~1e-7 relative) with the
// half-width squared padded by 1e-5 of its maximum and the interval widened
// by 2e-3 px plus 1e-5 relative — well above the fp32 rounding (about 1e-6
// of q) — then intersected with the effective rect (itself
// widened by a pixel). A cleared bit therefore never hides a composited
// pixel, and the blend warps skip the (entry, sub-tile) hits the rect test
// alone would admit.
constexpr int kMaskShift = 24;  // tile keys carry the mask above the tile id
constexpr uint32_t kTileIdMask = (1u << kMaskShift) - 1u;

struct MaskSplat {
  int4 er;                   // effective rect (pixels, widened by one)
  float mx, my, mxl, myl;    // mean2d as hi/lo pairs (dy must be accurate: q ~ q0 dy^2)
  float r, inv_ixx, q0;      // ixy / ixx, 1 / ixx, iyy - ixy^2 / ixx
  float qcut, pad;           // q threshold; 1e-5 * qcut / ixx
};

// rows = false: effective-rect test only (dsg_set_exact_masks; the parity
// tests check the two give bit-identical renders and gradients)
__device__ __forceinline__ uint32_t subtile_mask(const MaskSplat& sp, int ox, int oy, bool rows) {
  const int ry0 = max(sp.er.y, oy), ry1 = min(sp.er.w, oy + kTile - 1);
  const int cx0 = max(sp.er.x, ox), cx1 = min(sp.er.z, ox + kTile - 1);
  uint32_t m = 0;
  if (cx0 > cx1) return 0;
  if (!rows) {
    for (int y = ry0; y <= ry1; ++y) {
      const int sy = (y - oy) >> 2;
      if (cx0 < ox + 8) m |= 1u << (sy * 2);
      if (cx1 >= ox + 8) m |= 1u << (sy * 2 + 1);
    }
    return m;
  }
  const float mxh = sp.mx - 0.5f;  // exact (|mx| < 2^23): pixel x = centre - 0.5
  for (int y = ry0; y <= ry1; ++y) {
    const float dy = (((float)y + 0.5f) - sp.my) - sp.myl;
    const float h2 = (sp.qcut - dy * dy * sp.q0) * sp.inv_ixx + sp.pad;
    if (h2 < 0.f) continue;
    const float c = (mxh - sp.r * dy) + sp.mxl;  // row's minimum-q centre x, minus 0.5
    float h;  // MUFU sqrt: its ~1e-7 relative error is far inside the 1e-5 pad
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(h) : "f"(h2));
    // pixel x (centre x + 0.5) with centre in [c - h - eps, c + h + eps]
    const float t = h + (2.005e-3f + 1e-5f * (fabsf(c) + h));
    const float lo = ceilf(c - t), hi = floorf(c + t);
    const int xl = lo < (float)cx0 ? cx0 : (int)lo;
    const int xh = hi > (float)cx1 ? cx1 : (int)hi;
    if (xl > xh) continue;
    const int sy = (y - oy) >> 2;
    if (xl < ox + 8) m |= 1u << (sy * 2);
    if (xh >= ox + 8) m |= 1u << (sy * 2 + 1);
  }
  return m;
}

// K2: one (tile id, gaussian index) pair per overlapped tile, emitted in
// depth order; tile enumeration row-major inside the rect (render.hpp:127-133).
// The key's high byte carries the entry's sub-tile mask through the tile sort
// (the sort only ranks the tile-id bits).
__global__ void k_duplicate(const uint32_t* __restrict__ vis_idx, int64_t nv,
                            const uint32_t* __restrict__ offs, const int4* __restrict__ trect,
                            const int4* __restrict__ erect, const float4* __restrict__ rec,
                            const float4* __restrict__ mrow, bool rows, int tiles_x, int band_ty0,
                            int band_ty1, uint32_t* __restrict__ tile_key,
                            uint32_t* __restrict__ dup_val, uint32_t* __restrict__ dup_base) {
  DSG_PDL_ENTRY();
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nv) return;
  uint32_t i = vis_idx[s];
  uint32_t o = offs[s];
  if (dup_base) dup_base[i] = o;  // partial rows in emission (depth) order
  const int4 pr = trect[i];
  MaskSplat ms;
  ms.er = erect[i];
  {
    const float4 m0 = __ldg(rec + 3 * (size_t)i), k = __ldg(mrow + i);
    ms.mx = m0.x;
    ms.my = m0.y;
    ms.mxl = m0.z;
    ms.myl = m0.w;
    ms.r = k.x;
    ms.inv_ixx = k.y;
    ms.q0 = k.z;
    ms.qcut = k.w;
    ms.pad = 1e-5f * fabsf(k.w) * k.y;
  }
  const int4 r = make_int4(pr.x / kTile, max(pr.y / kTile, band_ty0), pr.z / kTile,
                           min(pr.w / kTile, band_ty1 - 1));
  for (int ty = r.y; ty <= r.w; ++ty)
    for (int tx = r.x; tx <= r.z; ++tx) {
      const uint32_t m = subtile_mask(ms, tx * kTile, ty * kTile, rows);
      tile_key[o] = (uint32_t)(ty * tiles_x + tx) | (m << kMaskShift);
      dup_val[o] = i;
      ++o;
    }
}

// K4: [start, end) of every tile in the sorted duplicate list, and the
// entries' sub-tile masks split off the keys (one coalesced byte per entry
// for the blend warps).
__global__ void k_tile_ranges(const uint32_t* __restrict__ tile_key, int64_t nd, uint2* ranges,
                              uint8_t* __restrict__ emask) {
  DSG_PDL_ENTRY();
  // four entries per thread: one 16 B key load, one 4 B mask store
  const int64_t e0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (e0 >= nd) return;
  uint32_t k[4];
  if (e0 + 4 <= nd) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(tile_key) + (e0 >> 2));
    k[0] = q.x; k[1] = q.y; k[2] = q.z; k[3] = q.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) k[j] = e0 + j < nd ? tile_key[e0 + j] : 0u;
  }
  uint32_t prev = e0 == 0 ? ~0u : (__ldg(tile_key + e0 - 1) & kTileIdMask);
  uint32_t m = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t e = e0 + j;
    if (e >= nd) break;
    const uint32_t t = k[j] & kTileIdMask;
    m |= (k[j] >> kMaskShift) << (8 * j);
    if (t != prev) {
      ranges[t].x = (uint32_t)e;
      if (e > 0) ranges[prev].y = (uint32_t)e;
    }
    prev = t;
  }
  if (e0 + 4 >= nd) ranges[prev].y = (uint32_t)nd;  // the last entry closes its tile
  if (e0 + 4 <= nd)
    *reinterpret_cast<uint32_t*>(emask + e0) = m;
  else
    for (int j = 0; e0 + j < nd; ++j) emask[e0 + j] = (uint8_t)(m >> (8 * j));
}

// Blend work units (blend.cu): tile i of the longest-first order gets
// ceil(len / seg_len) segments (at least one, so empty tiles still write the
// background); units of a tile are consecutive.
__global__ void k_unit_counts(const uint2* __restrict__ ranges, const uint32_t* __restrict__ order,
                              int nt, uint32_t seg, uint32_t* __restrict__ cnt) {
  DSG_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const uint2 r = ranges[order[i]];
  cnt[i] = max(1u, (r.y - r.x + seg - 1) / seg);
}

// Layout: unit i (< nt) = first segment of ordered tile i; segment k >= 1 of
// tile i = unit nt + (base[i] - i) + k - 1 (base[i] - i = later segments of
// earlier tiles); first_of maps a later unit back to its tile's first unit.
__global__ void k_unit_fill(const uint2* __restrict__ ranges, const uint32_t* __restrict__ order,
                            int nt, uint32_t seg, uint32_t split_len,
                            const uint32_t* __restrict__ base,
                            uint4* __restrict__ units, uint32_t* __restrict__ first_of) {
  DSG_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const uint32_t t = order[i];
  const uint2 r = ranges[t];
  const uint32_t b = base[i], nseg = base[i + 1] - b;
  // split: even the forward walks the segments in parallel (blend.cu)
  const uint32_t split = nseg > 1 && r.y - r.x > split_len ? 1u << 31 : 0u;
  for (uint32_t k = 0; k < nseg; ++k) {
    const uint32_t beg = r.x + k * seg, end = min(r.y, beg + seg);
    const uint32_t u = k == 0 ? (uint32_t)i : (uint32_t)nt + (b - i) + k - 1;
    units[u] = make_uint4(t, beg, end, k | (nseg << 16) | split);
    if (k > 0) first_of[u - nt] = (uint32_t)i;
  }
}

// Longest-first tile schedule for the blend kernels: tiles are bucketed by
// list length in quarter octaves (floor(4 log2 len)) and emitted heaviest
// bucket first, so the long lists start early instead of forming the tail
// (order inside a bucket is irrelevant: tiles are independent). Split lists
// (len > split_len) form the top bucket, so they are the first units (at
// most split_cap of them) and the split forward's per-tile grids cover them.
constexpr int kBins = 4 * 32 + 2;

__global__ void k_tile_bins(const uint2* __restrict__ ranges, int t0, int nt, uint32_t split,
                            uint32_t* bins, uint32_t* counts) {
  DSG_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const uint2 r = ranges[t0 + i];
  const uint32_t len = r.y - r.x;
  uint32_t b = 0;
  if (len > split) {
    b = kBins - 1;
  } else if (len) {
    const uint32_t e = 31u - __clz(len);                      // floor(log2 len)
    const uint32_t q = e >= 2 ? (len >> (e - 2)) & 3u : (len << (2 - e)) & 3u;
    b = 1u + 4u * e + q;                                      // 1 .. 128
  }
  bins[i] = b;
  atomicAdd(&counts[b], 1u);
}

__global__ void k_tile_bin_offsets(uint32_t* counts) {
  DSG_PDL_ENTRY();  // one warp: descending exclusive scan
  const int lane = threadIdx.x;
  uint32_t run = 0;
  for (int b = kBins - 1; b >= 0; --b) {
    const uint32_t c = counts[b];
    if (lane == 0) counts[b] = run;
    run += c;
  }
}

__global__ void k_tile_order(const uint32_t* __restrict__ bins, int t0, int nt, uint32_t* counts,
                             uint32_t* order) {
  DSG_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  order[atomicAdd(&counts[bins[i]], 1u)] = (uint32_t)(t0 + i);
}

inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Splats per tile row by projected centre (fp32; only balances the bands of
// the tile-parallel render, never decides a pixel). Block histograms in
// shared memory, then one global atomic per non-empty row.
__global__ void k_center_rows(const float* __restrict__ P, int64_t pitch, int64_t n, CamDev cam,
                              uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t h[];
  for (int t = threadIdx.x; t < cam.tiles_y; t += blockDim.x) h[t] = 0;
  __syncthreads();
  const float R0 = (float)cam.R[0], R1 = (float)cam.R[1], R2 = (float)cam.R[2];
  const float R3 = (float)cam.R[3], R4 = (float)cam.R[4], R5 = (float)cam.R[5];
  const float R6 = (float)cam.R[6], R7 = (float)cam.R[7], R8 = (float)cam.R[8];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float x = P[i] - (float)cam.pos[0], y = P[pitch + i] - (float)cam.pos[1],
                z = P[2 * pitch + i] - (float)cam.pos[2];
    const float tz = R6 * x + R7 * y + R8 * z;
    if (!(tz > (float)cam.near_plane)) continue;
    const float tx = R0 * x + R1 * y + R2 * z, ty = R3 * x + R4 * y + R5 * z;
    const float u = (float)cam.half_w + (float)cam.f * tx / tz;
    const float v = (float)cam.half_h - (float)cam.f * ty / tz;
    if (u < 0.f || u >= (float)cam.width || v < 0.f || v >= (float)cam.height) continue;
    atomicAdd(&h[min((int)v / kTile, cam.tiles_y - 1)], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < cam.tiles_y; t += blockDim.x)
    if (h[t]) atomicAdd(&hist[t], h[t]);
}

}  // namespace

void center_row_hist_dev(const float* params, int64_t pitch, int64_t n, const CamDev& cam,
                         uint32_t* hist, cudaStream_t st) {
  DSG_CUDA_CHECK(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * cam.tiles_y, st));
  if (n <= 0) return;
  const unsigned g = (unsigned)std::min<int64_t>(blocks(n, 256), 148 * 8);
  k_center_rows<<<g, 256, sizeof(uint32_t) * cam.tiles_y, st>>>(params, pitch, n, cam, hist);
  count_launch();
}

std::atomic<int> g_exact_masks{1};

void bin_frame(Frame& f, const float* params, int64_t pitch, int64_t n, const CamDev& cam,
               const RenderDev& rd, cudaStream_t st, StageTimer* timer) {
  StageTimer none;
  StageTimer& tm = timer ? *timer : none;
  tm.mark(0, st);
  f.n = n;
  f.tiles = (int64_t)cam.tiles_x * cam.tiles_y;
  f.rec.ensure(3 * (size_t)std::max<int64_t>(n, 1));
  f.trect.ensure(std::max<int64_t>(n, 1));
  f.erect.ensure(std::max<int64_t>(n, 1));
  f.mrow.ensure(std::max<int64_t>(n, 1));
  f.vslot.ensure(n + 1);
  f.tcount.ensure(std::max<int64_t>(n, 1));
  f.depth.ensure(std::max<int64_t>(n, 1));
  f.exact.ensure(3 * (size_t)std::max<int64_t>(n, 1));
  f.dup_base.ensure(std::max<int64_t>(n, 1) + 1);
  f.vis_key.ensure(std::max<int64_t>(n, 1));
  f.vis_idx.ensure(std::max<int64_t>(n, 1));
  f.vis_key2.ensure(std::max<int64_t>(n, 1));
  f.vis_idx2.ensure(std::max<int64_t>(n, 1));
  f.offs.ensure(std::max<int64_t>(n, 1) + 1);
  f.ranges.ensure(f.tiles);
  f.drange.ensure(2);
  DSG_CUDA_CHECK(cudaMemsetAsync(f.drange.get(), 0xff, sizeof(unsigned long long), st));  // min
  DSG_CUDA_CHECK(cudaMemsetAsync(f.drange.get() + 1, 0, sizeof(unsigned long long), st));  // max
  DSG_CUDA_CHECK(cudaMemsetAsync(f.ranges.get(), 0, f.tiles * sizeof(uint2), st));
  f.n_visible = 0;
  f.n_dup = 0;
  if (n > 0) {
    PreprocessArgs a;
    a.params = params;
    a.pitch = pitch;
    a.n = n;
    a.cam = cam;
    a.rd = rd;
    a.rec = f.rec.get();
    a.trect = f.trect.get();
    a.erect = f.erect.get();
    a.mrow = f.mrow.get();
    a.tcount = f.tcount.get();
    a.depth = f.depth.get();
    a.exact = f.exact.get();
    a.drange = f.drange.get();
    pdl_launch(k_preprocess, blocks(n, 256), 256, 0, st, a);
    count_launch();
    DSG_CUDA_CHECK(cudaGetLastError());
#if DSG_ROWS_BY_INDEX
    // Visible-slot scan, and the backward partial rows keyed by splat index
    // (K6 writes them, K7 reads them): row base of splat i = its tiles'
    // running count in index order, so K7's threads (consecutive splats)
    // read consecutive rows (chain + Adam 0.63 -> 0.58 ms). One dual pass.
    exclusive_scan_u32_dual(f.tcount.get(), f.vslot.get(), f.dup_base.get(), n, f.scan, st);
#else
    exclusive_scan_u32(f.tcount.get(), f.vslot.get(), n, f.scan, st, true);
#endif
    pdl_launch(k_vis_compact, blocks(n, 256), 256, 0, st, f.tcount.get(), f.depth.get(), f.drange.get(),
                                                  f.vslot.get(), n, f.vis_key.get(),
                                                  f.vis_idx.get());
    count_launch();
    tm.mark(1, st);
    uint32_t nvis = 0;
    DSG_CUDA_CHECK(cudaMemcpyAsync(&nvis, f.vslot.get() + n, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                   st));
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    f.n_visible = nvis;
  }
  const int64_t nv = f.n_visible;
  if (nv == 0) return;

  // depth sort of the visible set (stable; key = fp32 depth bits)
  bool alt = radix_sort_pairs<uint32_t>(f.vis_key.get(), f.vis_idx.get(), f.vis_key2.get(),
                                         f.vis_idx2.get(), nv, 0, kDepthKeyBits, f.sort, st, false);
  uint32_t* skey = alt ? f.vis_key2.get() : f.vis_key.get();
  uint32_t* sidx = alt ? f.vis_idx2.get() : f.vis_idx.get();
  uint32_t* runflag = alt ? f.vis_key.get() : f.vis_key2.get();  // free until k_gather_counts
  DSG_CUDA_CHECK(cudaMemsetAsync(runflag, 0, sizeof(uint32_t) * nv, st));
  constexpr uint32_t kLongCap = 1024;
  uint32_t* long_runs = f.long_runs.ensure(1 + 2 * kLongCap);
  DSG_CUDA_CHECK(cudaMemsetAsync(long_runs, 0, sizeof(uint32_t), st));
  pdl_launch(k_depth_mark, blocks(nv, 256), 256, 0, st, skey, sidx, nv, f.depth.get(), runflag);
  pdl_launch(k_depth_fixup, blocks(nv, 256), 256, 0, st, skey, sidx, nv, f.depth.get(), runflag,
                                                 long_runs, kLongCap);
  count_launch(2);
  tm.mark(2, st);
  f.sorted_idx = sidx;
  // per-splat tile counts in depth order, exclusive scan -> duplicate slots
  uint32_t* cnt = alt ? f.vis_key.get() : f.vis_key2.get();  // free buffer
  pdl_launch(k_gather_counts, blocks(nv, 256), 256, 0, st, sidx, nv, f.tcount.get(), cnt);
  count_launch();
  exclusive_scan_u32(cnt, f.offs.get(), nv, f.scan, st);
  uint32_t nd = 0, n_long = 0;
  DSG_CUDA_CHECK(cudaMemcpyAsync(&nd, f.offs.get() + nv, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaMemcpyAsync(&n_long, long_runs, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  if (n_long > kLongCap) {
    // very rare: more long near-coincident runs than the per-run path takes.
    // Sort the whole visible set by (fp64 depth bits, index) instead — the
    // reference comparator (render.hpp:98-101): depths are > near > 0, so
    // their bit patterns order as the values, and a stable sort of the
    // index-ordered compaction breaks ties by index.
    unsigned long long* rk = f.run_keys.ensure(2 * (size_t)nv);
    uint32_t* rv = f.run_vals.ensure(2 * (size_t)nv);
    pdl_launch(k_vis_compact, blocks(n, 256), 256, 0, st, f.tcount.get(), f.depth.get(), f.drange.get(),
                                                  f.vslot.get(), n, cnt, rv);
    k_run_keys<<<blocks(nv, 256), 256, 0, st>>>(rv, 0, (uint32_t)nv, f.depth.get(), rk, rv + nv);
    count_launch(2);
    const bool in_alt = radix_sort_pairs<uint64_t>(
        reinterpret_cast<uint64_t*>(rk), rv + nv, reinterpret_cast<uint64_t*>(rk) + nv, rv, nv, 0,
        64, f.sort, st);
    DSG_CUDA_CHECK(cudaMemcpyAsync(sidx, in_alt ? rv : rv + nv, sizeof(uint32_t) * nv,
                                   cudaMemcpyDeviceToDevice, st));
    pdl_launch(k_gather_counts, blocks(nv, 256), 256, 0, st, sidx, nv, f.tcount.get(), cnt);
    count_launch();
    exclusive_scan_u32(cnt, f.offs.get(), nv, f.scan, st);
  } else if (n_long > 0) {
    // rare: long runs of near-coincident depths with out-of-order pairs.
    // Radix-sort each by its fp64 depth bits, then redo the slots (the
    // duplicate total is order-independent).
    std::vector<uint32_t> runs(2 * n_long);
    DSG_CUDA_CHECK(cudaMemcpy(runs.data(), long_runs + 1, sizeof(uint32_t) * 2 * n_long,
                              cudaMemcpyDeviceToHost));
    for (uint32_t r = 0; r < n_long; ++r) {
      const uint32_t s0 = runs[2 * r], len = runs[2 * r + 1];
      unsigned long long* rk = f.run_keys.ensure(2 * (size_t)len);
      uint32_t* rv = f.run_vals.ensure(2 * (size_t)len);
      k_run_keys<<<blocks(len, 256), 256, 0, st>>>(sidx, s0, len, f.depth.get(), rk, rv);
      count_launch();
      const bool in_alt = radix_sort_pairs<uint64_t>(
          reinterpret_cast<uint64_t*>(rk), rv, reinterpret_cast<uint64_t*>(rk) + len, rv + len, len,
          0, 64, f.sort, st);
      DSG_CUDA_CHECK(cudaMemcpyAsync(sidx + s0, in_alt ? rv + len : rv, sizeof(uint32_t) * len,
                                     cudaMemcpyDeviceToDevice, st));
    }
    pdl_launch(k_gather_counts, blocks(nv, 256), 256, 0, st, sidx, nv, f.tcount.get(), cnt);
    count_launch();
    exclusive_scan_u32(cnt, f.offs.get(), nv, f.scan, st);
  }
  f.n_dup = nd;
  f.tile_key.ensure(std::max<uint32_t>(nd, 1));
  f.dup_val.ensure(std::max<uint32_t>(nd, 1));
  f.tile_key2.ensure(std::max<uint32_t>(nd, 1));
  f.dup_val2.ensure(std::max<uint32_t>(nd, 1));
  if (f.tiles > (int64_t)kTileIdMask) fail(kInvalidArgument, "image has too many tiles");
  pdl_launch(k_duplicate, blocks(nv, 256), 256, 0, st, sidx, nv, f.offs.get(), f.trect.get(),
                                               f.erect.get(), f.rec.get(), f.mrow.get(),
                                               g_exact_masks.load() != 0,
                                               cam.tiles_x, cam.band_ty0, cam.band_ty1,
                                               f.tile_key.get(), f.dup_val.get(),
                                               DSG_ROWS_BY_INDEX ? nullptr : f.dup_base.get());
  count_launch();
  tm.mark(3, st);
  int tile_bits = 1;
  while ((int64_t(1) << tile_bits) < f.tiles) ++tile_bits;
  bool alt2 = radix_sort_pairs<uint32_t>(f.tile_key.get(), f.dup_val.get(), f.tile_key2.get(),
                                          f.dup_val2.get(), nd, 0, tile_bits, f.sort, st, false);
  f.sorted_tile = alt2 ? f.tile_key2.get() : f.tile_key.get();
  f.sorted_val = alt2 ? f.dup_val2.get() : f.dup_val.get();
  f.emask.ensure(std::max<uint32_t>(nd, 1));
  pdl_launch(k_tile_ranges, blocks((nd + 3) / 4, 256), 256, 0, st, f.sorted_tile, nd, f.ranges.get(),
                                                 f.emask.get());
  count_launch();
  {
    const int t0 = cam.band_ty0 * cam.tiles_x;
    const int nt = (cam.band_ty1 - cam.band_ty0) * cam.tiles_x;
    f.tile_order.ensure(std::max(nt, 1));
    f.tile_bins.ensure(std::max(nt, 1) + kBins);
    uint32_t* counts = f.tile_bins.get() + std::max(nt, 1);
    DSG_CUDA_CHECK(cudaMemsetAsync(counts, 0, kBins * sizeof(uint32_t), st));
    // A frame whose tiles alone cannot fill the GPU (config 1: 256 tiles at
    // 256^2) gets shorter units and splits its long lists in the forward too;
    // a full frame keeps the forward's single walk (its dense tiles terminate
    // early, which the split forward cannot exploit).
    int dev = 0, sms = 148;
    DSG_CUDA_CHECK(cudaGetDevice(&dev));
    DSG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const bool underfilled = (int64_t)nt * 8 < (int64_t)sms * 4 * 28;  // 8 warps/tile
    f.seg_len = std::max<int64_t>(underfilled ? kSegMin / 2 : kSegMin,
                                  ((int64_t)nd + kSegDiv - 1) / kSegDiv);
    static const int64_t seg_env = [] {  // DSG_SEG_LEN: tuning override
      const char* e = std::getenv("DSG_SEG_LEN");
      return e ? std::max<int64_t>(std::atoll(e), 0) : int64_t(0);
    }();
    if (seg_env > 0) f.seg_len = seg_env;
    f.seg_len = (f.seg_len + 31) & ~int64_t(31);  // whole 32-entry chunks
    // forward splitting only for lists far beyond what termination usually
    // cuts short (the split forward re-walks later segments' products)
    f.split_len = underfilled ? kSplitFactor * f.seg_len
                              : std::max<int64_t>(kSplitMin, kSplitFactor * f.seg_len);
    static const int64_t split_env = [] {  // DSG_SPLIT_LEN: tuning override
      const char* e = std::getenv("DSG_SPLIT_LEN");
      return e ? std::max<int64_t>(std::atoll(e), 0) : int64_t(0);
    }();
    if (split_env > 0) f.split_len = std::max<int64_t>(split_env, f.seg_len);
    f.split_cap = (int64_t)nd > f.split_len ? (int64_t)nd / f.split_len + 1 : 0;
    pdl_launch(k_tile_bins, blocks(nt, 256), 256, 0, st, f.ranges.get(), t0, nt, (uint32_t)f.split_len,
                                                 f.tile_bins.get(), counts);
    pdl_launch(k_tile_bin_offsets, 1, 32, 0, st, counts);
    pdl_launch(k_tile_order, blocks(nt, 256), 256, 0, st, f.tile_bins.get(), t0, nt, counts,
                                                  f.tile_order.get());
    count_launch(3);
    // blend work units: ceil(len / seg_len) per tile in that order
    f.band_tiles = nt;
    f.unit_cap = nt + (int64_t)nd / f.seg_len + 1;
    f.units.ensure(f.unit_cap);
    f.unit_base.ensure(nt + 1);
    f.nonlast.ensure(std::max<int64_t>(f.unit_cap - nt, 1));
    f.ubuf.ensure((size_t)kUnitPlanes * f.unit_cap * kTile * kTile);
    uint32_t* ucnt = f.tile_bins.get();  // bins are consumed by k_tile_order
    pdl_launch(k_unit_counts, blocks(nt, 256), 256, 0, st, f.ranges.get(), f.tile_order.get(), nt,
                                                   (uint32_t)f.seg_len, ucnt);
    count_launch();
    exclusive_scan_u32(ucnt, f.unit_base.get(), nt, f.scan, st);
    pdl_launch(k_unit_fill, blocks(nt, 256), 256, 0, st, f.ranges.get(), f.tile_order.get(), nt,
                                                 (uint32_t)f.seg_len, (uint32_t)f.split_len,
                                                 f.unit_base.get(),
                                                 f.units.get(), f.nonlast.get());
    count_launch();
  }
  DSG_CUDA_CHECK(cudaGetLastError());
  tm.mark(4, st);
}

}  // namespace dsg
