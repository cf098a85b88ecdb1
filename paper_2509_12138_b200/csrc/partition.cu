// K10 slab partitioner and K12 ghost-trim merge compaction (sm_100a).
//
// partition_cloud (partition.hpp:42-104): the cut-axis coordinates become
// order-preserving u64 keys (with -0.0 folded onto +0.0, because the
// reference comparator treats them as equal) and are sorted stably with the
// onesweep sort, so the sorted order is (coordinate, index) exactly as the
// reference's std::sort comparator. Cuts are the fp64 midpoints of the
// neighbours at the count quantiles; ownership (half-open, outer slabs open)
// and ghost membership (distance to the finite owned interval <= margin) are
// flagged per partition and compacted in index order, so owned/ghost lists
// are bit-identical to the reference's.
//
// merge_models (partition.hpp:109-126): keep a splat iff its final mu is
// owned by its partition; order-preserving compaction of the planar model.
#include <cmath>
#include <limits>
#include <vector>

#include "dsg_internal.h"
#include "raster.h"

namespace dsg {

namespace {

__device__ __forceinline__ uint64_t ordered_key(double v) {
  if (v == 0.0) v = 0.0;  // -0.0 == +0.0 for the reference comparator
  uint64_t b = (uint64_t)__double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_axis_keys(const double* __restrict__ p, int64_t n, int axis, uint64_t* keys,
                            uint32_t* idx) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = ordered_key(p[3 * i + axis]);
  idx[i] = (uint32_t)i;
}

// Per point and partition: 1 = owned, 2 = ghost, 0 = neither (flags[k][i]).
__global__ void k_membership(const double* __restrict__ p, int64_t n, int axis, int nparts,
                             const double* __restrict__ cut_lo, const double* __restrict__ cut_hi,
                             const double* __restrict__ box_lo, const double* __restrict__ box_hi,
                             double margin, uint32_t* __restrict__ own,
                             uint32_t* __restrict__ ghost) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = p[3 * i + axis];
  for (int k = 0; k < nparts; ++k) {
    const bool o = v >= cut_lo[k] && v < cut_hi[k];
    bool g = false;
    if (!o) {
      const double lo = box_lo[k], hi = box_hi[k];
      const double d = v < lo ? lo - v : (v > hi ? v - hi : 0.0);
      g = d <= margin;
    }
    own[(int64_t)k * n + i] = o ? 1u : 0u;
    ghost[(int64_t)k * n + i] = g ? 1u : 0u;
  }
}

__global__ void k_compact(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                          int64_t n, uint32_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) out[pos[i]] = (uint32_t)i;
}

__global__ void k_merge_flags(const float* __restrict__ params, int64_t pitch, int64_t n, int axis,
                              double lo, double hi, uint32_t* __restrict__ flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = (double)params[axis * pitch + i];
  flag[i] = (v >= lo && v < hi) ? 1u : 0u;
}

__global__ void k_merge_scatter(const float* __restrict__ src, int64_t spitch, int64_t n,
                                const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                                float* __restrict__ dst, int64_t dpitch, int64_t dst_off) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  const int64_t o = dst_off + pos[i];
#pragma unroll
  for (int k = 0; k < kParams; ++k) dst[k * dpitch + o] = src[k * spitch + i];
}

inline unsigned nb(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + 255) / 256); }

}  // namespace

PartitionResult partition_dev(const double* host_pts, int64_t n, int nparts, double margin,
                              SortScratch& ss, ScanScratch& sc, cudaStream_t st) {
  if (n == 0) fail(kEmptyCloud, "cannot partition an empty cloud");
  if (nparts < 1) fail(kInvalidArgument, "partition count must be >= 1");
  if (nparts > n) fail(kInvalidArgument, "more partitions than points");
  if (margin < 0.0) fail(kInvalidArgument, "ghost margin must be >= 0");
  PartitionResult r;
  // Aabb of the cloud (pointcloud.hpp:25-30) and its longest axis (math.hpp:164-170)
  double lo[3] = {host_pts[0], host_pts[1], host_pts[2]}, hi[3] = {lo[0], lo[1], lo[2]};
  for (int64_t i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) {
      const double v = host_pts[3 * i + c];
      lo[c] = std::min(lo[c], v);
      hi[c] = std::max(hi[c], v);
    }
  const double e[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  const int axis = (e[0] >= e[1] && e[0] >= e[2]) ? 0 : (e[1] >= e[2] ? 1 : 2);
  r.axis = axis;
  DevBuf<double> pts;
  pts.ensure(3 * n);
  DSG_CUDA_CHECK(cudaMemcpyAsync(pts.get(), host_pts, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
  // stable sort by (coordinate, index)
  DevBuf<uint64_t> k1, k2;
  DevBuf<uint32_t> i1, i2;
  k1.ensure(n);
  k2.ensure(n);
  i1.ensure(n);
  i2.ensure(n);
  k_axis_keys<<<nb(n), 256, 0, st>>>(pts.get(), n, axis, k1.get(), i1.get());
  count_launch();
  bool alt = radix_sort_pairs<uint64_t>(k1.get(), i1.get(), k2.get(), i2.get(), n, 0, 64, ss, st);
  const uint32_t* sidx = alt ? i2.get() : i1.get();
  std::vector<uint32_t> ranks;
  for (int k = 1; k < nparts; ++k) {
    size_t rk = (size_t)n * (size_t)k / (size_t)nparts;
    ranks.push_back((uint32_t)(rk - 1));
    ranks.push_back((uint32_t)rk);
  }
  std::vector<double> cuts;
  for (size_t j = 0; j < ranks.size(); j += 2) {
    uint32_t a = 0, b = 0;
    DSG_CUDA_CHECK(cudaMemcpyAsync(&a, sidx + ranks[j], 4, cudaMemcpyDeviceToHost, st));
    DSG_CUDA_CHECK(cudaMemcpyAsync(&b, sidx + ranks[j + 1], 4, cudaMemcpyDeviceToHost, st));
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    cuts.push_back(0.5 * (host_pts[3 * (size_t)a + axis] + host_pts[3 * (size_t)b + axis]));
  }
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<double> clo(nparts), chi(nparts), blo(nparts), bhi(nparts);
  r.box.resize(6 * nparts);
  for (int k = 0; k < nparts; ++k) {
    clo[k] = k == 0 ? -inf : cuts[k - 1];
    chi[k] = k == nparts - 1 ? inf : cuts[k];
    double b[6] = {lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]};
    if (k > 0) b[axis] = cuts[k - 1];
    if (k < nparts - 1) b[3 + axis] = cuts[k];
    for (int c = 0; c < 6; ++c) r.box[6 * k + c] = b[c];
    blo[k] = b[axis];
    bhi[k] = b[3 + axis];
  }
  r.cut_lo = clo;
  r.cut_hi = chi;
  DevBuf<double> cd;
  cd.ensure(4 * nparts);
  std::vector<double> packed;
  packed.insert(packed.end(), clo.begin(), clo.end());
  packed.insert(packed.end(), chi.begin(), chi.end());
  packed.insert(packed.end(), blo.begin(), blo.end());
  packed.insert(packed.end(), bhi.begin(), bhi.end());
  DSG_CUDA_CHECK(cudaMemcpyAsync(cd.get(), packed.data(), sizeof(double) * 4 * nparts,
                                 cudaMemcpyHostToDevice, st));
  DevBuf<uint32_t> own, ghost, pos, out;
  own.ensure((size_t)nparts * n);
  ghost.ensure((size_t)nparts * n);
  pos.ensure(n + 1);
  out.ensure(n);
  k_membership<<<nb(n), 256, 0, st>>>(pts.get(), n, axis, nparts, cd.get(), cd.get() + nparts,
                                      cd.get() + 2 * nparts, cd.get() + 3 * nparts, margin,
                                      own.get(), ghost.get());
  count_launch();
  r.owned.resize(nparts);
  r.ghost.resize(nparts);
  for (int k = 0; k < nparts; ++k)
    for (int w = 0; w < 2; ++w) {
      const uint32_t* flag = (w == 0 ? own.get() : ghost.get()) + (size_t)k * n;
      exclusive_scan_u32(flag, pos.get(), n, sc, st);
      k_compact<<<nb(n), 256, 0, st>>>(flag, pos.get(), n, out.get());
      count_launch();
      uint32_t cnt = 0;
      DSG_CUDA_CHECK(cudaMemcpyAsync(&cnt, pos.get() + n, 4, cudaMemcpyDeviceToHost, st));
      DSG_CUDA_CHECK(cudaStreamSynchronize(st));
      std::vector<uint32_t>& dst = w == 0 ? r.owned[k] : r.ghost[k];
      dst.resize(cnt);
      if (cnt)
        DSG_CUDA_CHECK(cudaMemcpyAsync(dst.data(), out.get(), 4ull * cnt, cudaMemcpyDeviceToHost, st));
      DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    }
  return r;
}

void merge_trim_count(const MergeSrc* src, int np, int axis, MergeScratch& ms, ScanScratch& sc,
                      cudaStream_t st, int64_t* counts) {
  ms.base.assign(np + 1, 0);
  for (int k = 0; k < np; ++k) ms.base[k + 1] = ms.base[k] + src[k].n + 1;
  ms.flag.ensure(std::max<int64_t>(ms.base[np], 1));
  ms.pos.ensure(std::max<int64_t>(ms.base[np], 1));
  ms.cnt.ensure(std::max(np, 1));
  for (int k = 0; k < np; ++k) {
    const MergeSrc& s = src[k];
    uint32_t* pos = ms.pos.get() + ms.base[k];
    if (s.n > 0) {
      uint32_t* flag = ms.flag.get() + ms.base[k];
      k_merge_flags<<<nb(s.n), 256, 0, st>>>(s.params, s.pitch, s.n, axis, s.cut_lo, s.cut_hi, flag);
      count_launch();
      exclusive_scan_u32(flag, pos, s.n, sc, st);
      DSG_CUDA_CHECK(cudaMemcpyAsync(ms.cnt.get() + k, pos + s.n, 4, cudaMemcpyDeviceToDevice, st));
    } else {
      DSG_CUDA_CHECK(cudaMemsetAsync(ms.cnt.get() + k, 0, 4, st));
    }
  }
  std::vector<uint32_t> c(std::max(np, 1));
  DSG_CUDA_CHECK(cudaMemcpyAsync(c.data(), ms.cnt.get(), 4ull * np, cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  for (int k = 0; k < np; ++k) counts[k] = c[k];
}

void merge_trim_scatter(const MergeSrc& src, int k, MergeScratch& ms, float* dst, int64_t dpitch,
                        int64_t dst_off, cudaStream_t st) {
  if (src.n <= 0) return;
  k_merge_scatter<<<nb(src.n), 256, 0, st>>>(src.params, src.pitch, src.n,
                                             ms.flag.get() + ms.base[k], ms.pos.get() + ms.base[k],
                                             dst, dpitch, dst_off);
  count_launch();
}

}  // namespace dsg
