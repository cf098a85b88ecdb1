// Multi-GPU exchange: ghost-trim merge all-gather and the
// tile-parallel global render, over NCCL (NVLink 5 / NVSwitch).
//
// Training needs no collective (each GPU owns a slab partition). At the end:
//   1. each rank compacts the splats its partition owns (merge_models keep
//      rule, partition.hpp:120) on the device;
//   2. the survivor counts are all-gathered (int64);
//   3. the survivors are broadcast from every rank into one merged planar
//      model in (partition, index) order — merge_models' order
//      (partition.hpp:117-123) — so every GPU holds the merged model;
//   4. the merged model is rendered tile-parallel: rank r bins and blends
//      only its band of tile rows (preprocess is replicated), and the bands
//      are gathered to rank 0 with ncclSend/ncclRecv.
// NCCL is loaded with dlopen so the process shares whichever libnccl is
// already resident (e.g. torch's) instead of mapping a second copy.
#include <dlfcn.h>
#include <nccl.h>

#include <string>
#include <vector>

#include "dsg_internal.h"
#include "raster.h"

namespace dsg {

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  if (n.h) return n;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) fail(kWorkerFailure, std::string("cannot load NCCL: ") + dlerror());
  auto sym = [&](const char* s) {
    void* p = dlsym(h, s);
    if (!p) fail(kWorkerFailure, std::string("NCCL symbol missing: ") + s);
    return p;
  };
  n.GetUniqueId = (decltype(n.GetUniqueId))sym("ncclGetUniqueId");
  n.CommInitRank = (decltype(n.CommInitRank))sym("ncclCommInitRank");
  n.CommDestroy = (decltype(n.CommDestroy))sym("ncclCommDestroy");
  n.AllGather = (decltype(n.AllGather))sym("ncclAllGather");
  n.Broadcast = (decltype(n.Broadcast))sym("ncclBroadcast");
  n.Send = (decltype(n.Send))sym("ncclSend");
  n.Recv = (decltype(n.Recv))sym("ncclRecv");
  n.GroupStart = (decltype(n.GroupStart))sym("ncclGroupStart");
  n.GroupEnd = (decltype(n.GroupEnd))sym("ncclGroupEnd");
  n.GetErrorString = (decltype(n.GetErrorString))sym("ncclGetErrorString");
  n.h = h;
  return n;
}

void nc(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(kWorkerFailure, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

void nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  nc(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
}

void* nccl_comm_init(const uint8_t id_bytes[128], int nranks, int rank) {
  ncclUniqueId id;
  memcpy(&id, id_bytes, 128);
  ncclComm_t c = nullptr;
  nc(nccl().CommInitRank(&c, nranks, id, rank), "ncclCommInitRank");
  // NCCL connects lazily on first use: run one all-gather and one broadcast
  // per root now, so the timed merge does not pay connection setup.
  Nccl& N = nccl();
  DevBuf<float> tmp;
  tmp.ensure(2 * nranks + 2);
  cudaStream_t st;
  DSG_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  DSG_CUDA_CHECK(cudaMemsetAsync(tmp.get(), 0, sizeof(float) * (2 * nranks + 2), st));
  nc(N.AllGather(tmp.get() + 2 * nranks, tmp.get(), 1, ncclFloat32, c, st), "warm-up allgather");
  nc(N.GroupStart(), "group start");
  for (int r = 0; r < nranks; ++r)
    nc(N.Broadcast(tmp.get() + 2 * nranks + 1, tmp.get() + nranks + r, 1, ncclFloat32, r, c, st),
       "warm-up broadcast");
  nc(N.GroupEnd(), "group end");
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  DSG_CUDA_CHECK(cudaStreamDestroy(st));
  return c;
}

void nccl_comm_destroy(void* c) {
  if (c) nccl().CommDestroy((ncclComm_t)c);
}

// Steps 1-3 above. `merged` receives the merged model (reserved inside).
int64_t merge_allgather_dev(void* comm, int nranks, int rank, const ModelDev& local, int axis,
                            double cut_lo, double cut_hi, ModelDev& merged, ScanScratch& sc,
                            cudaStream_t st, float* wire_ms) {
  Nccl& N = nccl();
  ncclComm_t c = (ncclComm_t)comm;
  // 1. local compaction into a dense [14][cnt] buffer
  int64_t cnt = merge_compact_dev(local.params.get(), local.cap, local.n, axis, cut_lo, cut_hi,
                                  nullptr, 0, 0, sc, st);
  DevBuf<float> dense;
  dense.ensure((size_t)kParams * std::max<int64_t>(cnt, 1));
  merge_compact_dev(local.params.get(), local.cap, local.n, axis, cut_lo, cut_hi, dense.get(),
                    std::max<int64_t>(cnt, 1), 0, sc, st);
  // 2. counts
  DevBuf<int64_t> counts;
  counts.ensure(nranks + 1);
  DSG_CUDA_CHECK(cudaMemcpyAsync(counts.get() + nranks, &cnt, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  nc(N.AllGather(counts.get() + nranks, counts.get(), 1, ncclInt64, c, st), "allgather counts");
  std::vector<int64_t> hc(nranks);
  DSG_CUDA_CHECK(cudaMemcpyAsync(hc.data(), counts.get(), sizeof(int64_t) * nranks, cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  int64_t total = 0;
  std::vector<int64_t> off(nranks);
  for (int r = 0; r < nranks; ++r) {
    off[r] = total;
    total += hc[r];
  }
  // 3. every rank's survivors, broadcast row by row into the merged model
  merged.reserve(std::max<int64_t>(total, 1));
  merged.n = total;
  cudaEvent_t e0, e1;
  DSG_CUDA_CHECK(cudaEventCreate(&e0));
  DSG_CUDA_CHECK(cudaEventCreate(&e1));
  DSG_CUDA_CHECK(cudaEventRecord(e0, st));
  nc(N.GroupStart(), "group start");
  for (int r = 0; r < nranks; ++r) {
    if (hc[r] == 0) continue;
    for (int k = 0; k < kParams; ++k) {
      const float* send = r == rank ? dense.get() + (size_t)k * std::max<int64_t>(cnt, 1) : nullptr;
      nc(N.Broadcast(send, merged.params.get() + (size_t)k * merged.cap + off[r], (size_t)hc[r],
                     ncclFloat32, r, c, st),
         "broadcast survivors");
    }
  }
  nc(N.GroupEnd(), "group end");
  DSG_CUDA_CHECK(cudaEventRecord(e1, st));
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  float t = 0.f;
  DSG_CUDA_CHECK(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (wire_ms) *wire_ms = t;
  return total;
}

// Step 4: gather rank bands (tile rows [ty0_r, ty1_r)) of the planar image
// into rank 0's buffer.
void gather_bands_dev(void* comm, int nranks, int rank, float* rgb, int width, int height,
                      const std::vector<int>& row0, const std::vector<int>& row1, cudaStream_t st) {
  Nccl& N = nccl();
  ncclComm_t c = (ncclComm_t)comm;
  const int64_t npix = (int64_t)width * height;
  nc(N.GroupStart(), "group start");
  for (int r = 1; r < nranks; ++r) {
    const int64_t p0 = (int64_t)row0[r] * width;
    const int64_t cntp = (int64_t)(row1[r] - row0[r]) * width;
    if (cntp <= 0) continue;
    for (int ch = 0; ch < 3; ++ch) {
      float* p = rgb + ch * npix + p0;
      if (rank == 0) nc(N.Recv(p, (size_t)cntp, ncclFloat32, r, c, st), "recv band");
      else if (rank == r) nc(N.Send(p, (size_t)cntp, ncclFloat32, 0, c, st), "send band");
    }
  }
  nc(N.GroupEnd(), "group end");
}

}  // namespace dsg
