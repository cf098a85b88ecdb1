// Warp/block scan helpers (shuffle based), used by the sort, scan and
// compaction kernels.
#pragma once
#include <stdint.h>

namespace dsg {

template <class T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// Exclusive block-wide sum over NT threads (NT multiple of 32, <= 1024).
// smem: >= 33 elements (per-warp prefixes in [0, 32), the total in [32]).
// Returns the exclusive prefix; *aggregate = total. Ends with a
// __syncthreads so smem can be reused.
template <int NT, class T>
__device__ __forceinline__ T block_exclusive_sum(T v, T* aggregate, T* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  T inc = warp_inclusive_sum(v);
  if (lane == 31) smem[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < NW ? smem[lane] : T(0);
    T wi = warp_inclusive_sum(w);
    if (lane < NW) smem[lane] = wi - w;
    if (lane == NW - 1) smem[32] = wi;  // not [31]: with 32 warps that is warp 31's prefix
  }
  __syncthreads();
  T r = smem[warp] + inc - v;
  *aggregate = smem[32];
  __syncthreads();
  return r;
}

}  // namespace dsg
