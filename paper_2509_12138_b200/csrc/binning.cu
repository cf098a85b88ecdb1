// K1 preprocess, depth-sort fix-up, K2 duplicate, K4 tile ranges (sm_100a).
//
// K1 replaces try_project (projection.hpp:24-57) and the cull/rect part of
// prepare_splats (render.hpp:62-97). Every integer- or order-producing value
// (camera-space depth, mean2d, cov2d, pixel rect, culling) is computed in
// exact fp64 without FMA contraction, so rects, tile counts and the sorted
// key lists match the x86-64 reference bit-for-bit; the blend payload is
// stored as fp32 (mean2d as a hi/lo pair so pixel offsets stay exact).
//
// Ordering: visible splats are sorted by fp32 depth bits (monotone in the
// fp64 depth), runs of equal fp32 keys are re-ordered by (fp64 depth, index)
// — the reference comparator (render.hpp:98-101) — and the duplicates are
// then stably sorted by tile id, so every tile list is in reference
// compositing order.
#include <atomic>

#include "dsg_internal.h"
#include "raster.h"
#include "scan_util.cuh"

namespace dsg {

namespace {

__global__ void __launch_bounds__(256) k_preprocess(PreprocessArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  bool vis = false;
  float depth_f = 0.f;
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
        const double q_eff = fmin(a.rd.sigma_sq, 2.0 * log(op / a.rd.alpha_cutoff));
        {  // sub-tile mask constants (see subtile_mask): ixy/ixx, 1/ixx, q0, qcut
          const double inv = 1.0 / ixx, rr = ixy * inv;
          a.mrow[i] = make_float4((float)rr, (float)inv, (float)(iyy - ixy * rr),
                                  (float)(q_eff + 1e-9 * fabs(q_eff) + 1e-12));
        }
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
        depth_f = (float)pr.depth;
        vis = true;
      }
    }
    a.tcount[i] = count;
  }
  // warp-aggregated compaction of the visible set (order fixed by the sort)
  uint32_t mask = __ballot_sync(0xffffffffu, vis);
  uint32_t base = 0;
  if (mask != 0 && lane == __ffs(mask) - 1) base = atomicAdd(a.vis_count, (uint32_t)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, mask != 0 ? __ffs(mask) - 1 : 0);
  if (vis) {
    uint32_t slot = base + __popc(mask & ((1u << lane) - 1u));
    a.vis_key[slot] = __float_as_uint(depth_f);
    a.vis_idx[slot] = (uint32_t)i;
  }
  // key range of the visible set: the depth sort only needs the bits of
  // (key - min), typically 24 of 32 (3 radix passes instead of 4)
  uint32_t kmin = vis ? __float_as_uint(depth_f) : 0xffffffffu;
  uint32_t kmax = vis ? __float_as_uint(depth_f) : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  // one pair of atomics per block, and only when it can move the bound
  // (same-address atomics from every warp serialise in L2)
  __shared__ uint32_t smin[8], smax[8];
  const int warp = threadIdx.x >> 5;
  if (lane == 0) {
    smin[warp] = kmin;
    smax[warp] = kmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      kmin = min(kmin, smin[w]);
      kmax = max(kmax, smax[w]);
    }
    volatile uint32_t* c = a.vis_count;
    if (kmin < c[1]) atomicMin(a.vis_count + 1, kmin);
    if (kmax > c[2]) atomicMax(a.vis_count + 2, kmax);
  }
}

// Re-order runs of equal fp32 depth keys by (fp64 depth, index): the
// reference comparator (render.hpp:98-101). Runs are tiny; insertion sort.
__global__ void k_depth_fixup(const uint32_t* __restrict__ key, uint32_t* idx, int64_t n,
                              const double* __restrict__ depth) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  uint32_t k = key[s];
  if (s > 0 && key[s - 1] == k) return;          // not a run start
  if (s + 1 >= n || key[s + 1] != k) return;     // singleton
  int64_t e = s + 1;
  while (e < n && key[e] == k) ++e;
  for (int64_t j = s + 1; j < e; ++j) {
    uint32_t v = idx[j];
    double dv = depth[v];
    int64_t m = j - 1;
    while (m >= s) {
      uint32_t u = idx[m];
      double du = depth[u];
      if (du < dv || (du == dv && u < v)) break;
      idx[m + 1] = u;
      --m;
    }
    idx[m + 1] = v;
  }
}

__global__ void k_gather_counts(const uint32_t* __restrict__ vis_idx, int64_t nv,
                                const uint32_t* __restrict__ tcount, uint32_t* out) {
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
// formed by K1 from the fp64 values (qcut = q_eff + 1e-9 relative); per row they are evaluated
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
  for (int y = ry0; y <= ry1; ++y) {
    const float dy = (((float)y + 0.5f) - sp.my) - sp.myl;
    const float h2 = (sp.qcut - dy * dy * sp.q0) * sp.inv_ixx + sp.pad;
    if (h2 < 0.f) continue;
    const float c = (sp.mx - sp.r * dy) + sp.mxl;  // x of the row's minimum q
    const float h = sqrtf(h2);
    const float eps = 2e-3f + 1e-5f * (fabsf(c) + h);
    // pixel x (centre x + 0.5) with centre in [c - h - eps, c + h + eps]
    const float lo = ceilf(c - h - eps - 0.5f), hi = floorf(c + h + eps - 0.5f);
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
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nv) return;
  uint32_t i = vis_idx[s];
  uint32_t o = offs[s];
  dup_base[i] = o;
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
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nd) return;
  const uint32_t k = tile_key[e];
  const uint32_t t = k & kTileIdMask;
  emask[e] = (uint8_t)(k >> kMaskShift);
  if (e == 0 || (tile_key[e - 1] & kTileIdMask) != t) ranges[t].x = (uint32_t)e;
  if (e == nd - 1 || (tile_key[e + 1] & kTileIdMask) != t) ranges[t].y = (uint32_t)(e + 1);
}

// Longest-first tile schedule for the blend kernels: tiles are bucketed by
// floor(log2(list length)) and emitted heaviest bucket first, so the long
// lists start early instead of forming the tail (order inside a bucket is
// irrelevant: tiles are independent).
__global__ void k_tile_bins(const uint2* __restrict__ ranges, int t0, int nt, uint32_t* bins,
                            uint32_t* counts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const uint2 r = ranges[t0 + i];
  const uint32_t len = r.y - r.x;
  const uint32_t b = len ? 32u - __clz(len) : 0u;  // 0..32
  bins[i] = b;
  atomicAdd(&counts[b], 1u);
}

__global__ void k_tile_bin_offsets(uint32_t* counts) {  // one warp: descending exclusive scan
  const int lane = threadIdx.x;
  uint32_t run = 0;
  for (int b = 32; b >= 0; --b) {
    const uint32_t c = counts[b];
    if (lane == 0) counts[b] = run;
    run += c;
  }
}

__global__ void k_tile_order(const uint32_t* __restrict__ bins, int t0, int nt, uint32_t* counts,
                             uint32_t* order) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  order[atomicAdd(&counts[bins[i]], 1u)] = (uint32_t)(t0 + i);
}

inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

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
  f.tcount.ensure(std::max<int64_t>(n, 1));
  f.depth.ensure(std::max<int64_t>(n, 1));
  f.exact.ensure(3 * (size_t)std::max<int64_t>(n, 1));
  f.dup_base.ensure(std::max<int64_t>(n, 1));
  f.vis_key.ensure(std::max<int64_t>(n, 1));
  f.vis_idx.ensure(std::max<int64_t>(n, 1));
  f.vis_key2.ensure(std::max<int64_t>(n, 1));
  f.vis_idx2.ensure(std::max<int64_t>(n, 1));
  f.offs.ensure(std::max<int64_t>(n, 1) + 1);
  f.ranges.ensure(f.tiles);
  f.counters.ensure(4);
  DSG_CUDA_CHECK(cudaMemsetAsync(f.counters.get(), 0, 4 * sizeof(uint32_t), st));
  DSG_CUDA_CHECK(cudaMemsetAsync(f.counters.get() + 1, 0xff, sizeof(uint32_t), st));  // key min
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
    a.vis_key = f.vis_key.get();
    a.vis_idx = f.vis_idx.get();
    a.vis_count = f.counters.get();
    k_preprocess<<<blocks(n, 256), 256, 0, st>>>(a);
    count_launch();
    DSG_CUDA_CHECK(cudaGetLastError());
    tm.mark(1, st);
    uint32_t c3[3] = {0, 0, 0};
    DSG_CUDA_CHECK(cudaMemcpyAsync(c3, f.counters.get(), 3 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    f.n_visible = c3[0];
    f.key_min = c3[1];
    f.key_max = c3[2];
  }
  const int64_t nv = f.n_visible;
  if (nv == 0) return;
  int depth_bits = 1;
  while (depth_bits < 32 && ((uint64_t)(f.key_max - f.key_min) >> depth_bits) != 0) ++depth_bits;
  // depth sort of the visible set (stable; key = fp32 depth bits)
  bool alt = radix_sort_pairs<uint32_t>(f.vis_key.get(), f.vis_idx.get(), f.vis_key2.get(),
                                         f.vis_idx2.get(), nv, 0, depth_bits, f.sort, st,
                                         f.key_min, false);
  uint32_t* skey = alt ? f.vis_key2.get() : f.vis_key.get();
  uint32_t* sidx = alt ? f.vis_idx2.get() : f.vis_idx.get();
  k_depth_fixup<<<blocks(nv, 256), 256, 0, st>>>(skey, sidx, nv, f.depth.get());
  count_launch();
  tm.mark(2, st);
  f.sorted_idx = sidx;
  // per-splat tile counts in depth order, exclusive scan -> duplicate slots
  uint32_t* cnt = alt ? f.vis_key.get() : f.vis_key2.get();  // free buffer
  k_gather_counts<<<blocks(nv, 256), 256, 0, st>>>(sidx, nv, f.tcount.get(), cnt);
  count_launch();
  exclusive_scan_u32(cnt, f.offs.get(), nv, f.scan, st);
  uint32_t nd = 0;
  DSG_CUDA_CHECK(cudaMemcpyAsync(&nd, f.offs.get() + nv, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  f.n_dup = nd;
  f.tile_key.ensure(std::max<uint32_t>(nd, 1));
  f.dup_val.ensure(std::max<uint32_t>(nd, 1));
  f.tile_key2.ensure(std::max<uint32_t>(nd, 1));
  f.dup_val2.ensure(std::max<uint32_t>(nd, 1));
  if (f.tiles > (int64_t)kTileIdMask) fail(kInvalidArgument, "image has too many tiles");
  k_duplicate<<<blocks(nv, 256), 256, 0, st>>>(sidx, nv, f.offs.get(), f.trect.get(),
                                               f.erect.get(), f.rec.get(), f.mrow.get(),
                                               g_exact_masks.load() != 0,
                                               cam.tiles_x, cam.band_ty0, cam.band_ty1,
                                               f.tile_key.get(), f.dup_val.get(),
                                               f.dup_base.get());
  count_launch();
  tm.mark(3, st);
  int tile_bits = 1;
  while ((int64_t(1) << tile_bits) < f.tiles) ++tile_bits;
  bool alt2 = radix_sort_pairs<uint32_t>(f.tile_key.get(), f.dup_val.get(), f.tile_key2.get(),
                                          f.dup_val2.get(), nd, 0, tile_bits, f.sort, st, 0u,
                                          false);
  f.sorted_tile = alt2 ? f.tile_key2.get() : f.tile_key.get();
  f.sorted_val = alt2 ? f.dup_val2.get() : f.dup_val.get();
  f.emask.ensure(std::max<uint32_t>(nd, 1));
  k_tile_ranges<<<blocks(nd, 256), 256, 0, st>>>(f.sorted_tile, nd, f.ranges.get(),
                                                 f.emask.get());
  count_launch();
  {
    const int t0 = cam.band_ty0 * cam.tiles_x;
    const int nt = (cam.band_ty1 - cam.band_ty0) * cam.tiles_x;
    f.tile_order.ensure(std::max(nt, 1));
    f.tile_bins.ensure(std::max(nt, 1) + 33);
    uint32_t* counts = f.tile_bins.get() + std::max(nt, 1);
    DSG_CUDA_CHECK(cudaMemsetAsync(counts, 0, 33 * sizeof(uint32_t), st));
    k_tile_bins<<<blocks(nt, 256), 256, 0, st>>>(f.ranges.get(), t0, nt, f.tile_bins.get(), counts);
    k_tile_bin_offsets<<<1, 32, 0, st>>>(counts);
    k_tile_order<<<blocks(nt, 256), 256, 0, st>>>(f.tile_bins.get(), t0, nt, counts,
                                                  f.tile_order.get());
    count_launch(3);
  }
  DSG_CUDA_CHECK(cudaGetLastError());
  tm.mark(4, st);
}

}  // namespace dsg
