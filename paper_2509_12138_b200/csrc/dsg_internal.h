// Host-side internals of libdsg: device buffers, contexts, models, launchers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "dsg_common.cuh"

namespace dsg {

// Error raised inside the library and mapped to a C-ABI status at the
// boundary. code is dsplat::ErrorCode (error.hpp:10-31).
struct Error {
  int code;
  std::string msg;
};
enum Code {
  kBehindCamera = 0, kInvalidRig, kUnknownKind, kIsovalueOutOfRange, kEmptyCloud,
  kDimensionMismatch, kTooSmall, kEmptyBand, kEmptyInterior, kMismatchedCounts, kNoViews,
  kStaleForward, kIoError, kMalformedFile, kWorkerFailure, kTimeout, kManifestMismatch,
  kMissingBaseline, kInvalidArgument
};
[[noreturn]] void fail(int code, const std::string& msg);
// Counts this library's kernel launches (reported by bench.py as gpu_launches).
void count_launch(int n = 1);

// Growable raw device allocation (never shrinks; contents not preserved).
template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
  T* ensure(size_t n) {
    if (n > cap) {
      release();
      size_t c = n + n / 4 + 64;
      DSG_CUDA_CHECK(cudaMalloc(&ptr, c * sizeof(T)));
      cap = c;
    }
    return ptr;
  }
  T* get() const { return ptr; }
  void swap(DevBuf& o) {
    std::swap(ptr, o.ptr);
    std::swap(cap, o.cap);
  }
};

// Scratch for the radix sort and scans.
struct SortScratch {
  DevBuf<uint32_t> hist;      // [passes][256] digit histograms, then exclusive scans
  DevBuf<uint32_t> status;    // [passes][parts][256] look-back words
  DevBuf<uint32_t> counters;  // [passes] partition tickets
  std::vector<uint32_t> host_hist;
};

struct ScanScratch {
  DevBuf<uint32_t> block_sums;
};

// Stable LSD radix sort of (keys, vals) on key bits [begin_bit, end_bit),
// onesweep style: one global-histogram pass over the keys, then one
// decoupled-look-back scatter kernel per 8-bit digit. Ping-pongs between
// (keys, vals) and (keys_alt, vals_alt); returns true when the sorted result
// ends in the *_alt buffers. Digits whose histogram is a single bin are
// skipped (stable no-op). Synchronizes the stream once (histogram readback).
// With skip_trivial = false every pass runs and the call never synchronizes
// (the per-step sorts, whose digits all vary).
template <class K>
bool radix_sort_pairs(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, int64_t n,
                      int begin_bit, int end_bit, SortScratch& s, cudaStream_t st,
                      bool skip_trivial = true);

// Exclusive prefix sum of n u32 into out (out[n] = total). out may alias in.
// flags: sum (in[i] != 0) instead of in[i] (order-preserving compaction).
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, ScanScratch& s,
                        cudaStream_t st, bool flags = false);
// Both scans of one input in one pass: out_flags = scan of (in[i] != 0),
// out_vals = scan of in[i] (each with the total at [n]; totals < 2^32).
void exclusive_scan_u32_dual(const uint32_t* in, uint32_t* out_flags, uint32_t* out_vals,
                             int64_t n, ScanScratch& s, cudaStream_t st);

}  // namespace dsg
