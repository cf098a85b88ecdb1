// Onesweep LSD radix sort and exclusive scan (sm_100a).
//
// Replaces the reference's std::sort by (depth, index) (render.hpp:98-101)
// and the std::vector push_back binning (render.hpp:117-135): the raster
// pipeline sorts visible splats by depth once, duplicates them per tile in
// that order, then sorts the duplicates stably by tile id with this kernel,
// which reproduces the reference's per-tile compositing order exactly.
//
// Per digit pass: each CTA takes a ticket (partition id), loads 256x12 keys
// warp-striped (coalesced), ranks them per digit with warp match/popc in input
// order (stable), publishes its digit counts with a 2-bit flag in one 32-bit
// word, looks back over earlier partitions to form its exclusive digit
// prefix, stages the keys digit-sorted in shared memory and writes them out
// in coalesced runs. The global digit bases come from one histogram pass.
#include "dsg_internal.h"
#include "scan_util.cuh"

namespace dsg {

namespace {

constexpr int kRadixBits = 8;
constexpr int kRadix = 256;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
#ifndef DSG_SORT_ITEMS
#define DSG_SORT_ITEMS 12  // with 3 CTAs/SM: -6% depth sort against 16 and 2 (round 2 A/B)
#endif
constexpr int kSortItems = DSG_SORT_ITEMS;
#ifndef DSG_LOOKBACK
#define DSG_LOOKBACK 16
#endif
constexpr int kLookback = DSG_LOOKBACK;
constexpr int kPart = kSortThreads * kSortItems;  // keys per partition
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagPrefix = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <class K>
__global__ void __launch_bounds__(256) k_digit_hist(const K* __restrict__ keys, int64_t n,
                                                    int begin_bit, int passes,
                                                    uint32_t* __restrict__ ghist) {
  DSG_PDL_ENTRY();
  // 4 copies (one per warp pair) of up to 8 passes x 256 bins. Each thread
  // counts runs of equal digits in registers and flushes a run with one
  // shared atomic: high digits of sort keys are nearly constant, so this
  // removes the same-address contention that serialises per-key atomics.
  constexpr int kCopies = 4;
  __shared__ uint32_t h[kCopies][8][kRadix];
  for (int i = threadIdx.x; i < kCopies * 8 * kRadix; i += blockDim.x) (&h[0][0][0])[i] = 0;
  __syncthreads();
  const int cp = (threadIdx.x >> 5) & (kCopies - 1);
  uint32_t cur[8], cnt[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    cur[p] = 0;
    cnt[p] = 0;
  }
  auto count = [&](const K k) {
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      if (p >= passes) break;
      const uint32_t d = (uint32_t)((k >> (begin_bit + kRadixBits * p)) & (kRadix - 1));
      if (d != cur[p] && cnt[p]) {
        atomicAdd(&h[cp][p][cur[p]], cnt[p]);
        cnt[p] = 0;
      }
      cur[p] = d;
      ++cnt[p];
    }
  };
  int64_t i0 = 0;
  if constexpr (sizeof(K) == 4) {
    if ((reinterpret_cast<uintptr_t>(keys) & 15) != 0) goto scalar;
    // 32-bit keys: four per thread per step (16 B loads, the warp reads
    // 512 contiguous bytes), four times fewer dependent load round trips
    const int64_t n4 = n / 4;
    const uint4* k4 = reinterpret_cast<const uint4*>(keys);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
      const uint4 q = __ldg(k4 + i);
      count((K)q.x);
      count((K)q.y);
      count((K)q.z);
      count((K)q.w);
    }
    i0 = n4 * 4;
  }
scalar:
  for (int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    count(keys[i]);
#pragma unroll
  for (int p = 0; p < 8; ++p)
    if (p < passes && cnt[p]) atomicAdd(&h[cp][p][cur[p]], cnt[p]);
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
    const int p = i / kRadix, d = i % kRadix;
    uint32_t v = 0;
#pragma unroll
    for (int c = 0; c < kCopies; ++c) v += h[c][p][d];
    if (v) atomicAdd(&ghist[i], v);
  }
}

// Exclusive scan of each pass's 256 bins (one block per pass).
__global__ void k_hist_scan(uint32_t* ghist) {
  DSG_PDL_ENTRY();
  __shared__ uint32_t tmp[33];
  uint32_t* h = ghist + blockIdx.x * kRadix;
  uint32_t agg;
  uint32_t ex = block_exclusive_sum<kRadix>(h[threadIdx.x], &agg, tmp);
  h[threadIdx.x] = ex;
}

template <class K>
struct OnesweepSmem {
  uint32_t warp_hist[kSortWarps][kRadix];
  uint32_t block_excl[kRadix];
  uint32_t global_base[kRadix];
  K keys[kPart];       // the partition as loaded (TMA), then digit-sorted for the store
  uint32_t vals[kPart];
  uint64_t bar;        // mbarrier of the bulk loads
  uint32_t part;
  uint32_t scan[33];
};

#ifndef DSG_SORT_TMA
#define DSG_SORT_TMA 1
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// 1-D bulk copy global -> shared (TMA engine), completion counted in bytes
// on an mbarrier; dst, src and bytes 16 B aligned.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}

template <class K>
#ifndef DSG_SORT_MINB
#define DSG_SORT_MINB 3  // 3 CTAs/SM at 12 keys per thread, no spills
#endif
__global__ void __launch_bounds__(kSortThreads, DSG_SORT_MINB) k_onesweep(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
    uint32_t* __restrict__ vout, int64_t n, int shift,
    const uint32_t* __restrict__ gscan, uint32_t* status, uint32_t* counter) {
  DSG_PDL_ENTRY();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  OnesweepSmem<K>& sm = *reinterpret_cast<OnesweepSmem<K>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if DSG_SORT_TMA
  // The partition's keys and values arrive by two bulk copies (TMA) into the
  // staging arrays the digit-sorted store uses later; one thread issues
  // them as soon as the ticket is drawn, the rest zero the histograms.
  const bool tma = ((reinterpret_cast<uintptr_t>(kin) | reinterpret_cast<uintptr_t>(vin)) & 15) == 0;
  if (tid == 0) {
    const uint32_t part0 = atomicAdd(counter, 1u);
    sm.part = part0;
    if (tma) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sm.bar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      const int64_t b0 = (int64_t)part0 * kPart;
      const int64_t c0 = n - b0 < kPart ? n - b0 : (int64_t)kPart;
      const uint32_t kb = (uint32_t)(c0 * sizeof(K)) & ~15u, vb = (uint32_t)(c0 * 4) & ~15u;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&sm.bar)),
                   "r"(kb + vb)
                   : "memory");
      if (kb) bulk_load(sm.keys, kin + b0, kb, &sm.bar);
      if (vb) bulk_load(sm.vals, vin + b0, vb, &sm.bar);
    }
  }
#else
  const bool tma = false;
  if (tid == 0) sm.part = atomicAdd(counter, 1u);
#endif
  for (int i = tid; i < kSortWarps * kRadix; i += kSortThreads) (&sm.warp_hist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t part = sm.part;
  const int64_t base = (int64_t)part * kPart;
  const int count = n - base < kPart ? (int)(n - base) : kPart;

  K k[kSortItems];
  uint32_t v[kSortItems];
  uint32_t dig[kSortItems];
  uint32_t rank[kSortItems];
  const int wloc = warp * 32 * kSortItems;
  if (tma) {
    // the tail past the last whole 16 B of a short final partition
    const int kt = (int)(((uint32_t)(count * sizeof(K)) & ~15u) / sizeof(K));
    const int vt = (int)(((uint32_t)(count * 4) & ~15u) / 4);
    for (int j = kt + tid; j < count; j += kSortThreads) sm.keys[j] = kin[base + j];
    for (int j = vt + tid; j < count; j += kSortThreads) sm.vals[j] = vin[base + j];
    mbar_wait(&sm.bar, 0);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
      const int j = wloc + i * 32 + lane;
      const bool valid = j < count;
      k[i] = valid ? sm.keys[j] : K(0);
      v[i] = valid ? sm.vals[j] : 0u;
      dig[i] = valid ? (uint32_t)((k[i] >> shift) & (kRadix - 1)) : 0x100u;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
      const int j = wloc + i * 32 + lane;
      const bool valid = j < count;
      k[i] = valid ? kin[base + j] : K(0);
      v[i] = valid ? vin[base + j] : 0u;
      dig[i] = valid ? (uint32_t)((k[i] >> shift) & (kRadix - 1)) : 0x100u;
    }
  }
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    uint32_t d = dig[i];
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t before = d < kRadix ? sm.warp_hist[warp][d] : 0u;
    __syncwarp();
    if (d < kRadix && (__ffs(peers) - 1) == lane) sm.warp_hist[warp][d] = before + __popc(peers);
    __syncwarp();
    rank[i] = before + __popc(peers & lt);
  }
  __syncthreads();

  // Thread d owns digit d: exclusive offsets across warps, block total,
  // published at once so later partitions can sum past this one.
  const int d = tid;
  uint32_t total = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) {
    uint32_t c = sm.warp_hist[w][d];
    sm.warp_hist[w][d] = total;
    total += c;
  }
  volatile uint32_t* vs = status;
  vs[(size_t)part * kRadix + d] = (part == 0 ? kFlagPrefix : kFlagAgg) | total;
  uint32_t bagg;
  uint32_t bex = block_exclusive_sum<kSortThreads>(total, &bagg, sm.scan);
  sm.block_excl[d] = bex;
  __syncthreads();

  // Stage the partition digit-sorted in shared memory: only block-local
  // offsets are needed, so this happens before the look-back, which then
  // runs with the key registers dead (a wider window without spills) and
  // gives the predecessors more time to publish their prefixes.
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    uint32_t dg = dig[i];
    if (dg < kRadix) {
      uint32_t pos = sm.block_excl[dg] + sm.warp_hist[warp][dg] + rank[i];
      sm.keys[pos] = k[i];
      sm.vals[pos] = v[i];
    }
  }

  // Decoupled look-back over earlier partitions for this digit.
  uint32_t excl = 0;
  if (part != 0) {
    int64_t p = (int64_t)part - 1;
    // read kLookback predecessors per round trip (partition 0 always holds a
    // prefix): the first wave of resident partitions otherwise walks back
    // through hundreds of aggregates one L2 round trip at a time
    while (true) {
      uint32_t s[kLookback];
#pragma unroll
      for (int j = 0; j < kLookback; ++j) {
        s[j] = 2u << 30;  // kFlagPrefix, total 0: before partition 0
        if (p - j >= 0) s[j] = vs[(size_t)(p - j) * kRadix + d];
      }
      int j = 0;
      bool done = false;
#pragma unroll
      for (; j < kLookback; ++j) {
        const uint32_t flag = s[j] & ~kValueMask;
        if (flag == 0) break;  // not published yet: resume from p - j
        excl += s[j] & kValueMask;
        if (flag == kFlagPrefix) {
          done = true;
          break;
        }
      }
      if (done) break;
      p -= j;
    }
    vs[(size_t)part * kRadix + d] = kFlagPrefix | (excl + total);
  }
  sm.global_base[d] = gscan[d] + excl;
  __syncthreads();
  for (int j = tid; j < count; j += kSortThreads) {
    K key = sm.keys[j];
    uint32_t dg = (uint32_t)((key >> shift) & (kRadix - 1));
    uint32_t out = sm.global_base[dg] + (uint32_t)j - sm.block_excl[dg];
    kout[out] = key;
    vout[out] = sm.vals[j];
  }
}

// ---- exclusive scan (reduce, scan block sums, downsweep) ---------------------
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t* __restrict__ in,
                                                              int64_t n, uint32_t* sums,
                                                              bool flags) {
  DSG_PDL_ENTRY();
  __shared__ uint32_t tmp[33];
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + (int64_t)i * kScanThreads + threadIdx.x;
    if (idx < n) s += flags ? (uint32_t)(in[idx] != 0) : in[idx];
  }
  uint32_t agg;
  block_exclusive_sum<kScanThreads>(s, &agg, tmp);
  s = agg;
  if (threadIdx.x == 0) sums[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) k_scan_sums(uint32_t* sums, int64_t nb) {
  DSG_PDL_ENTRY();
  __shared__ uint32_t tmp[33];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += 1024) {
    int64_t i = base + threadIdx.x;
    uint32_t v = i < nb ? sums[i] : 0u, agg;
    uint32_t ex = block_exclusive_sum<1024>(v, &agg, tmp);
    if (i < nb) sums[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[nb] = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(const uint32_t* __restrict__ in,
                                                            uint32_t* out, int64_t n,
                                                            const uint32_t* __restrict__ sums,
                                                            bool flags) {
  DSG_PDL_ENTRY();
  __shared__ uint32_t tmp[33];
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t local = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? (flags ? (uint32_t)(in[base + i] != 0) : in[base + i]) : 0u;
    local += v[i];
  }
  uint32_t agg;
  uint32_t run = block_exclusive_sum<kScanThreads>(local, &agg, tmp);
  uint32_t ex[kScanItems];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    ex[i] = run;
    run += v[i];
  }
  uint32_t off = sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) out[base + i] = ex[i] + off;
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = sums[gridDim.x];
}

// Dual scan: (in[i] != 0) and in[i] summed together as one u64, the flag
// count in the high word (the low word's running sum never exceeds the u32
// total, so it never carries).
using u64 = unsigned long long;
__device__ __forceinline__ u64 pack2(uint32_t v) { return ((u64)(v != 0) << 32) | v; }

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce2(const uint32_t* __restrict__ in,
                                                               int64_t n, u64* sums) {
  DSG_PDL_ENTRY();
  __shared__ u64 tmp[33];
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + (int64_t)i * kScanThreads + threadIdx.x;
    if (idx < n) s += pack2(in[idx]);
  }
  u64 agg;
  block_exclusive_sum<kScanThreads>(s, &agg, tmp);
  if (threadIdx.x == 0) sums[blockIdx.x] = agg;
}

__global__ void __launch_bounds__(1024) k_scan_sums2(u64* sums, int64_t nb) {
  DSG_PDL_ENTRY();
  __shared__ u64 tmp[33];
  __shared__ u64 carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += 1024) {
    int64_t i = base + threadIdx.x;
    u64 v = i < nb ? sums[i] : 0ull, agg;
    u64 ex = block_exclusive_sum<1024>(v, &agg, tmp);
    if (i < nb) sums[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[nb] = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down2(const uint32_t* __restrict__ in,
                                                             uint32_t* out_f, uint32_t* out_v,
                                                             int64_t n, const u64* __restrict__ sums) {
  DSG_PDL_ENTRY();
  __shared__ u64 tmp[33];
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  u64 local = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? in[base + i] : 0u;
    local += pack2(v[i]);
  }
  u64 agg;
  u64 run = block_exclusive_sum<kScanThreads>(local, &agg, tmp) + sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) {
      out_f[base + i] = (uint32_t)(run >> 32);
      out_v[base + i] = (uint32_t)run;
    }
    run += pack2(v[i]);
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    out_f[n] = (uint32_t)(sums[gridDim.x] >> 32);
    out_v[n] = (uint32_t)sums[gridDim.x];
  }
}

}  // namespace

void exclusive_scan_u32_dual(const uint32_t* in, uint32_t* out_flags, uint32_t* out_vals,
                             int64_t n, ScanScratch& s, cudaStream_t st) {
  if (n <= 0) {
    DSG_CUDA_CHECK(cudaMemsetAsync(out_flags, 0, sizeof(uint32_t), st));
    DSG_CUDA_CHECK(cudaMemsetAsync(out_vals, 0, sizeof(uint32_t), st));
    return;
  }
  int64_t nb = (n + kScanTile - 1) / kScanTile;
  u64* sums = reinterpret_cast<u64*>(s.block_sums.ensure(2 * (nb + 1)));
  pdl_launch(k_scan_reduce2, (unsigned)nb, kScanThreads, 0, st, in, n, sums);
  pdl_launch(k_scan_sums2, 1, 1024, 0, st, sums, nb);
  pdl_launch(k_scan_down2, (unsigned)nb, kScanThreads, 0, st, in, out_flags, out_vals, n,
             (const u64*)sums);
  count_launch(3);
  DSG_CUDA_CHECK(cudaGetLastError());
}

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, ScanScratch& s,
                        cudaStream_t st, bool flags) {
  if (n <= 0) {
    DSG_CUDA_CHECK(cudaMemsetAsync(out, 0, sizeof(uint32_t), st));
    return;
  }
  int64_t nb = (n + kScanTile - 1) / kScanTile;
  uint32_t* sums = s.block_sums.ensure(nb + 1);
  pdl_launch(k_scan_reduce, (unsigned)nb, kScanThreads, 0, st, in, n, sums, flags);
  count_launch();
  pdl_launch(k_scan_sums, 1, 1024, 0, st, sums, nb);
  count_launch();
  pdl_launch(k_scan_down, (unsigned)nb, kScanThreads, 0, st, in, out, n, sums, flags);
  count_launch();
  DSG_CUDA_CHECK(cudaGetLastError());
}

template <class K>
bool radix_sort_pairs(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, int64_t n,
                      int begin_bit, int end_bit, SortScratch& s, cudaStream_t st,
                      bool skip_trivial) {
  if (n <= 1 || end_bit <= begin_bit) return false;
  if (n > (int64_t)kValueMask) fail(kInvalidArgument, "radix sort: too many keys");
  const int passes = (end_bit - begin_bit + kRadixBits - 1) / kRadixBits;
  const int64_t parts = (n + kPart - 1) / kPart;
  uint32_t* hist = s.hist.ensure((size_t)passes * kRadix);
  uint32_t* status = s.status.ensure((size_t)passes * parts * kRadix);
  uint32_t* counters = s.counters.ensure(passes);
  DSG_CUDA_CHECK(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * passes * kRadix, st));
  DSG_CUDA_CHECK(cudaMemsetAsync(status, 0, sizeof(uint32_t) * passes * parts * kRadix, st));
  DSG_CUDA_CHECK(cudaMemsetAsync(counters, 0, sizeof(uint32_t) * passes, st));
  int hist_blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  pdl_launch(k_digit_hist<K>, hist_blocks, 256, 0, st, keys, n, begin_bit, passes, hist);
  count_launch();
  // Which digits actually vary? (a single populated bin = identity pass)
  std::vector<bool> trivial(passes, false);
  if (skip_trivial) {
    s.host_hist.resize((size_t)passes * kRadix);
    DSG_CUDA_CHECK(cudaMemcpyAsync(s.host_hist.data(), hist, sizeof(uint32_t) * passes * kRadix,
                                   cudaMemcpyDeviceToHost, st));
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    for (int p = 0; p < passes; ++p)
      for (int d = 0; d < kRadix; ++d)
        if (s.host_hist[(size_t)p * kRadix + d] == (uint32_t)n) trivial[p] = true;
  }
  pdl_launch(k_hist_scan, passes, kRadix, 0, st, hist);
  count_launch();
  const size_t smem = sizeof(OnesweepSmem<K>);
  DSG_CUDA_CHECK(cudaFuncSetAttribute(k_onesweep<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  bool in_alt = false;
  for (int p = 0; p < passes; ++p) {
    if (trivial[p]) continue;
    const K* ki = in_alt ? keys_alt : keys;
    const uint32_t* vi = in_alt ? vals_alt : vals;
    K* ko = in_alt ? keys : keys_alt;
    uint32_t* vo = in_alt ? vals : vals_alt;
    pdl_launch(k_onesweep<K>, (unsigned)parts, kSortThreads, smem, st, ki, vi, ko, vo, n, begin_bit + kRadixBits * p, hist + (size_t)p * kRadix,
        status + (size_t)p * parts * kRadix, counters + p);
    count_launch();
    in_alt = !in_alt;
  }
  DSG_CUDA_CHECK(cudaGetLastError());
  return in_alt;
}

template bool radix_sort_pairs<uint32_t>(uint32_t*, uint32_t*, uint32_t*, uint32_t*, int64_t, int,
                                         int, SortScratch&, cudaStream_t, bool);
template bool radix_sort_pairs<uint64_t>(uint64_t*, uint32_t*, uint64_t*, uint32_t*, int64_t, int,
                                         int, SortScratch&, cudaStream_t, bool);

}  // namespace dsg
