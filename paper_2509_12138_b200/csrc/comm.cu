// Multi-GPU exchange: ghost-trim merge all-gather and the
// tile-parallel global render, over NCCL (NVLink 5 / NVSwitch).
//
// Training needs no collective (each GPU owns a slab partition). At the end:
//   1. each rank compacts the splats its partition owns (merge_models keep
//      rule, partition.hpp:120) on the device;
//   2. the survivor counts are all-gathered (int64);
//   3. the survivors are all-gathered as packed 56 B records (one NCCL
//      all-gather per partition round, padded to the largest slab) and
//      scattered into one merged planar model in (partition, index) order —
//      merge_models' order (partition.hpp:117-123) — so every GPU holds the
//      merged model (peer-memory pull / push / copy variants beside it);
//   4. the merged model is rendered tile-parallel: rank r bins and blends
//      only its band of tile rows (preprocess is replicated), and the bands
//      are gathered to rank 0 with ncclSend/ncclRecv.
// NCCL is loaded with dlopen so the process shares whichever libnccl is
// already resident (e.g. torch's) instead of mapping a second copy.
#include <dlfcn.h>
#include <cstdlib>
#include <cstring>
#include <nccl.h>

#include <mutex>
#include <string>
#include <vector>

#include "dsg_internal.h"
#include "raster.h"

namespace dsg {

const char* g_merge_path = "none";  // last merge exchange: "peer" or "nccl"

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // optional (NCCL >= 2.19): buffer registration
  ncclResult_t (*CommRegister)(const ncclComm_t, void*, size_t, void**) = nullptr;
  ncclResult_t (*CommDeregister)(const ncclComm_t, void*) = nullptr;
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
  n.AllReduce = (decltype(n.AllReduce))sym("ncclAllReduce");
  n.Send = (decltype(n.Send))sym("ncclSend");
  n.Recv = (decltype(n.Recv))sym("ncclRecv");
  n.GroupStart = (decltype(n.GroupStart))sym("ncclGroupStart");
  n.GroupEnd = (decltype(n.GroupEnd))sym("ncclGroupEnd");
  n.GetErrorString = (decltype(n.GetErrorString))sym("ncclGetErrorString");
  n.CommInitRankConfig = (decltype(n.CommInitRankConfig))dlsym(h, "ncclCommInitRankConfig");
  n.CommSplit = (decltype(n.CommSplit))dlsym(h, "ncclCommSplit");
  n.CommRegister = (decltype(n.CommRegister))dlsym(h, "ncclCommRegister");
  n.CommDeregister = (decltype(n.CommDeregister))dlsym(h, "ncclCommDeregister");
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
  // 64 CTAs per collective (NCCL's default caps them at 32): the merge's
  // all-gather of 0.75 GB per rank moves 493 instead of 442 GB/s into each
  // GPU at N = 4 (tools/merge_bw.py; 48: 424, 96: 466, 128: 463).
  // DSG_NCCL_CTAS overrides (0 = NCCL's default).
  static const int ctas = [] {
    const char* e = std::getenv("DSG_NCCL_CTAS");
    return e ? std::atoi(e) : 64;
  }();
  if (ctas > 0 && nccl().CommInitRankConfig) {
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.minCTAs = ctas;
    cfg.maxCTAs = ctas;
    nc(nccl().CommInitRankConfig(&c, nranks, id, rank, &cfg), "ncclCommInitRankConfig");
  } else {
    nc(nccl().CommInitRank(&c, nranks, id, rank), "ncclCommInitRank");
  }
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

// Exchange buffers registered with the communicator (ncclCommRegister), kept
// per communicator and grown on demand: 501 vs 493 GB/s into each GPU at N = 4
// with 64 CTAs (NCCL-allocated cuMem buffers were slower: 407).
// DSG_NCCL_REG=0 falls back to per-call plain buffers.
struct RegBuf {
  void* ptr = nullptr;
  void* handle = nullptr;
  size_t bytes = 0;
};
struct CommBufs {
  void* comm = nullptr;
  RegBuf send, recv;
};
static std::vector<CommBufs>& comm_bufs() {
  static std::vector<CommBufs> v;
  return v;
}
static std::mutex& comm_bufs_mu() {
  static std::mutex m;
  return m;
}
static bool reg_on() {
  static const bool on = [] {
    const char* e = std::getenv("DSG_NCCL_REG");
    return !(e && e[0] == '0');
  }();
  return on;
}
static void reg_free(Nccl& N, void* comm, RegBuf& b) {
  if (!b.ptr) return;
  if (b.handle) N.CommDeregister((ncclComm_t)comm, b.handle);
  cudaFree(b.ptr);
  b = RegBuf{};
}
static bool reg_ensure(Nccl& N, void* comm, RegBuf& b, size_t bytes) {
  if (b.ptr && b.bytes >= bytes) return true;
  reg_free(N, comm, b);
  if (cudaMalloc(&b.ptr, bytes) != cudaSuccess) {
    cudaGetLastError();
    b = RegBuf{};
    return false;
  }
  b.bytes = bytes;
  if (N.CommRegister((ncclComm_t)comm, b.ptr, bytes, &b.handle) != ncclSuccess) b.handle = nullptr;
  return true;
}
// send/recv of at least the given sizes for `comm`, or false (plain buffers then)
static bool exchange_buffers(void* comm, size_t send_bytes, size_t recv_bytes, float** send,
                             float** recv) {
  Nccl& N = nccl();
  if (!reg_on() || !N.CommRegister || !N.CommDeregister) return false;
  std::lock_guard<std::mutex> lk(comm_bufs_mu());
  CommBufs* cb = nullptr;
  for (auto& x : comm_bufs())
    if (x.comm == comm) cb = &x;
  if (!cb) {
    comm_bufs().push_back(CommBufs{comm, {}, {}});
    cb = &comm_bufs().back();
  }
  if (!reg_ensure(N, comm, cb->send, send_bytes) || !reg_ensure(N, comm, cb->recv, recv_bytes))
    return false;
  *send = (float*)cb->send.ptr;
  *recv = (float*)cb->recv.ptr;
  return true;
}

// A second communicator over the same ranks with NCCL's default CTA count,
// for the band gather's send/recv (64 CTAs slow those small transfers down:
// RT 4K render 3.5 -> 4.3 ms at N = 4). Collective; null when the library
// has no ncclCommSplit.
void* nccl_comm_split_default(void* comm, int rank) {
  Nccl& N = nccl();
  if (!comm || !N.CommSplit) return nullptr;
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;  // explicit: a split may inherit the parent's
  cfg.minCTAs = 1;
  cfg.maxCTAs = 32;
  ncclComm_t out = nullptr;
  nc(N.CommSplit((ncclComm_t)comm, 0, rank, &out, &cfg), "ncclCommSplit");
  return out;
}

void nccl_comm_destroy(void* c) {
  if (!c) return;
  Nccl& N = nccl();
  std::lock_guard<std::mutex> lk(comm_bufs_mu());
  auto& v = comm_bufs();
  for (size_t i = 0; i < v.size(); ++i)
    if (v[i].comm == c) {
      reg_free(N, c, v[i].send);
      reg_free(N, c, v[i].recv);
      v.erase(v.begin() + (long)i);
      break;
    }
  N.CommDestroy((ncclComm_t)c);
}

namespace {
// survivors, planar [14][pitch] -> packed records [cnt][14] (56 B per splat)
__global__ void k_pack_records(const float* __restrict__ dense, int64_t pitch, int64_t cnt,
                               float* __restrict__ rec) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt * kParams) return;
  const int64_t i = t / kParams;
  const int k = (int)(t - i * kParams);
  rec[t] = dense[k * pitch + i];
}
// the gathered [R][maxc][14] records -> merged planar model, rank r's
// survivors at offset off[r] (merge_models' (partition, index) order)
__global__ void k_unpack_records(const float* __restrict__ rec, int64_t maxc, int nranks,
                                 const int64_t* __restrict__ cnt, const int64_t* __restrict__ off,
                                 float* __restrict__ P, int64_t pitch) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)nranks * maxc * kParams) return;
  const int64_t row = t / kParams;
  const int k = (int)(t - row * kParams);
  const int r = (int)(row / maxc);
  const int64_t i = row - (int64_t)r * maxc;
  if (i >= cnt[r]) return;  // padding
  P[k * pitch + off[r] + i] = rec[t];
}
// Push one local partition's survivors (dense planar [14][cnt]) into every
// rank's merged planar model at the partition's offset: blockIdx.y = the
// destination rank, reached through its CUDA IPC mapping over NVLink.
// Reads and writes are coalesced per plane; all destinations are written
// concurrently, so every link carries traffic at once.
__global__ void __launch_bounds__(256) k_peer_push(const float* __restrict__ dense, int64_t dpitch,
                                                   int64_t cnt, float* const* __restrict__ dst,
                                                   const int64_t* __restrict__ dst_pitch,
                                                   int64_t off) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  float* d = dst[blockIdx.y];
  const int64_t pitch = dst_pitch[blockIdx.y];
#pragma unroll
  for (int c = 0; c < kParams; ++c) d[c * pitch + off + i] = __ldg(dense + c * dpitch + i);
}

// Pull: one launch over every partition (blockIdx.y = partition k), each
// block copying 256 records of partition k from the owning GPU's packed
// buffer (CUDA IPC mapping, NVLink reads of 16 B) through shared memory into
// the local merged planar store — all peers' links busy at once.
#ifndef DSG_PEER_RECS
#define DSG_PEER_RECS 1024  // records per block: 14 float4 NVLink loads in flight per thread
#endif
constexpr int kPeerRecs = DSG_PEER_RECS;
struct PullPart {
  const float* src;  // partition's first record on its owner
  int64_t cnt, off;
};
__global__ void __launch_bounds__(256) k_peer_pull(const PullPart* __restrict__ parts,
                                                   float* __restrict__ P, int64_t pitch) {
  extern __shared__ float4 sm4[];  // kPeerRecs * kParams floats
  float* sm = reinterpret_cast<float*>(sm4);
  const PullPart pp = parts[blockIdx.y];
  const int64_t b0 = (int64_t)blockIdx.x * kPeerRecs;
  if (b0 >= pp.cnt) return;
  const int nrec = (int)(pp.cnt - b0 < kPeerRecs ? pp.cnt - b0 : (int64_t)kPeerRecs);
  const float4* s4 = reinterpret_cast<const float4*>(pp.src + b0 * kParams);
  const int nf4 = (nrec * kParams + 3) / 4;  // sources are padded to whole float4s
  constexpr int kPer = (kPeerRecs * kParams / 4 + 255) / 256;
  float4 v[kPer];  // issue every load before the first store
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int i = threadIdx.x + u * 256;
    if (i < nf4) v[u] = s4[i];
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int i = threadIdx.x + u * 256;
    if (i < nf4) sm4[i] = v[u];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nrec * kParams; i += blockDim.x) {
    const int c = i / nrec, r = i - c * nrec;
    P[c * pitch + pp.off + b0 + r] = sm[r * kParams + c];
  }
}
}  // namespace

// Peer-memory variants of step 3 (DSG_MERGE_PATH=push / copy; the NCCL
// all-gather is the default, measured fastest on the 4-GPU box: DESIGN §7):
// every rank publishes the CUDA IPC handle and pitch of its merged model's
// parameter store (a 72 B all-gather), maps the others', and pushes each of
// its partitions' survivors straight into every rank's merged model at the
// partition's offset — k_peer_push (the transfer and the planar placement in
// one kernel, all destinations at once) or copy-engine plane copies. A
// one-word all-reduce after the pushes tells every rank its merged model is
// complete.
static bool merge_push_peers(Nccl& N, ncclComm_t c, int nranks, int rank, int nlocal,
                             const std::deque<DevBuf<float>>& dense,
                             const std::vector<int64_t>& cnt, const std::vector<int64_t>& off,
                             ModelDev& merged, cudaStream_t st, float* wire_ms,
                             bool copy_engines = false) {
  struct Pub {
    cudaIpcMemHandle_t h;
    int64_t pitch;
  };
  static_assert(sizeof(Pub) == 72, "published record");
  Pub mine;
  std::memset(&mine, 0, sizeof mine);
  mine.pitch = merged.cap;
  bool ok = cudaIpcGetMemHandle(&mine.h, merged.params.get()) == cudaSuccess;
  if (!ok) cudaGetLastError();  // still take part in the collectives: all ranks decide together
  DevBuf<uint8_t> pbuf;
  pbuf.ensure(sizeof(Pub) * (nranks + 1));
  DSG_CUDA_CHECK(cudaMemcpyAsync(pbuf.get() + sizeof(Pub) * nranks, &mine, sizeof(Pub),
                                 cudaMemcpyHostToDevice, st));
  nc(N.AllGather(pbuf.get() + sizeof(Pub) * nranks, pbuf.get(), sizeof(Pub), ncclUint8, c, st),
     "allgather handles");
  std::vector<Pub> pubs(nranks);
  DSG_CUDA_CHECK(cudaMemcpyAsync(pubs.data(), pbuf.get(), sizeof(Pub) * nranks,
                                 cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  std::vector<float*> dst(nranks, nullptr);
  std::vector<int64_t> pitch(nranks);
  for (int r = 0; r < nranks; ++r) {
    pitch[r] = pubs[r].pitch;
    if (r == rank) {
      dst[r] = merged.params.get();
      continue;
    }
    if (!ok) continue;
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, pubs[r].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = false;
      continue;
    }
    dst[r] = static_cast<float*>(p);
  }
  DevBuf<int> flag;
  flag.ensure(1);
  const int okv = ok ? 1 : 0;
  DSG_CUDA_CHECK(cudaMemcpyAsync(flag.get(), &okv, sizeof(int), cudaMemcpyHostToDevice, st));
  nc(N.AllReduce(flag.get(), flag.get(), 1, ncclInt32, ncclMin, c, st), "allreduce ipc status");
  int all_ok = 0;
  DSG_CUDA_CHECK(cudaMemcpyAsync(&all_ok, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  if (all_ok) {
    DevBuf<float*> dptr;
    DevBuf<int64_t> dpitch;
    dptr.ensure(nranks);
    dpitch.ensure(nranks);
    DSG_CUDA_CHECK(cudaMemcpyAsync(dptr.get(), dst.data(), sizeof(float*) * nranks,
                                   cudaMemcpyHostToDevice, st));
    DSG_CUDA_CHECK(cudaMemcpyAsync(dpitch.get(), pitch.data(), sizeof(int64_t) * nranks,
                                   cudaMemcpyHostToDevice, st));
    cudaEvent_t e0, e1;
    DSG_CUDA_CHECK(cudaEventCreate(&e0));
    DSG_CUDA_CHECK(cudaEventCreate(&e1));
    DSG_CUDA_CHECK(cudaEventRecord(e0, st));
    if (copy_engines) {
      // plane segments copied by the copy engines, one stream per destination
      std::vector<cudaStream_t> ss(nranks);
      std::vector<cudaEvent_t> done(nranks);
      for (int r = 0; r < nranks; ++r) {
        DSG_CUDA_CHECK(cudaStreamCreateWithFlags(&ss[r], cudaStreamNonBlocking));
        DSG_CUDA_CHECK(cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming));
        DSG_CUDA_CHECK(cudaStreamWaitEvent(ss[r], e0, 0));
      }
      for (int j = 0; j < nlocal; ++j) {
        const int k = j * nranks + rank;
        if (cnt[k] == 0) continue;
        for (int r = 0; r < nranks; ++r)
          for (int ch = 0; ch < kParams; ++ch)
            DSG_CUDA_CHECK(cudaMemcpyAsync(dst[r] + ch * pitch[r] + off[k],
                                           dense[j].get() + ch * std::max<int64_t>(cnt[k], 1),
                                           sizeof(float) * cnt[k], cudaMemcpyDeviceToDevice,
                                           ss[r]));
      }
      for (int r = 0; r < nranks; ++r) {
        DSG_CUDA_CHECK(cudaEventRecord(done[r], ss[r]));
        DSG_CUDA_CHECK(cudaStreamWaitEvent(st, done[r], 0));
      }
      DSG_CUDA_CHECK(cudaEventRecord(e1, st));
      DSG_CUDA_CHECK(cudaStreamSynchronize(st));
      for (int r = 0; r < nranks; ++r) {
        cudaEventDestroy(done[r]);
        cudaStreamDestroy(ss[r]);
      }
    } else {
      for (int j = 0; j < nlocal; ++j) {
        const int k = j * nranks + rank;
        if (cnt[k] == 0) continue;
        const dim3 grid((unsigned)((cnt[k] + 255) / 256), (unsigned)nranks);
        k_peer_push<<<grid, 256, 0, st>>>(dense[j].get(), std::max<int64_t>(cnt[k], 1), cnt[k],
                                          dptr.get(), dpitch.get(), off[k]);
        count_launch();
      }
      DSG_CUDA_CHECK(cudaEventRecord(e1, st));
    }
    // every rank's pushes have landed before anyone uses its merged model
    nc(N.AllReduce(flag.get(), flag.get(), 1, ncclInt32, ncclMin, c, st), "allreduce done");
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    float t = 0.f;
    DSG_CUDA_CHECK(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (wire_ms) *wire_ms = t;
  }
  for (int r = 0; r < nranks; ++r)
    if (r != rank && dst[r]) cudaIpcCloseMemHandle(dst[r]);
  return all_ok != 0;
}

// Pull variant: every rank packs its partitions' survivors into one buffer
// of 56 B records (each partition padded to an even count, so record starts
// are 16 B aligned), publishes its IPC handle, and pulls all partitions it
// does not own with one k_peer_pull launch.
static bool merge_pull_peers(Nccl& N, ncclComm_t c, int nranks, int rank, int nlocal,
                             const std::deque<DevBuf<float>>& dense,
                             const std::vector<int64_t>& cnt, const std::vector<int64_t>& off,
                             ModelDev& merged, cudaStream_t st, float* wire_ms) {
  const int P = nranks * nlocal;
  auto padded = [&](int k) { return (cnt[k] + 1) & ~int64_t(1); };
  std::vector<int64_t> roff(P, 0);  // record offset of partition k in its owner's buffer
  for (int r = 0; r < nranks; ++r) {
    int64_t o = 0;
    for (int j = 0; j < nlocal; ++j) {
      roff[j * nranks + r] = o;
      o += padded(j * nranks + r);
    }
  }
  int64_t mine_recs = 0;
  for (int j = 0; j < nlocal; ++j) mine_recs += padded(j * nranks + rank);
  DevBuf<float> send;
  send.ensure((size_t)std::max<int64_t>(mine_recs, 2) * kParams + 4);
  for (int j = 0; j < nlocal; ++j) {
    const int k = j * nranks + rank;
    if (cnt[k] > 0) {
      k_pack_records<<<(unsigned)((cnt[k] * kParams + 255) / 256), 256, 0, st>>>(
          dense[j].get(), std::max<int64_t>(cnt[k], 1), cnt[k], send.get() + roff[k] * kParams);
      count_launch();
    }
  }
  cudaIpcMemHandle_t mine;
  std::memset(&mine, 0, sizeof mine);
  bool ok = cudaIpcGetMemHandle(&mine, send.get()) == cudaSuccess;
  if (!ok) cudaGetLastError();
  DevBuf<uint8_t> hbuf;
  hbuf.ensure((size_t)64 * (nranks + 1));
  DSG_CUDA_CHECK(cudaMemcpyAsync(hbuf.get() + 64 * nranks, &mine, 64, cudaMemcpyHostToDevice, st));
  nc(N.AllGather(hbuf.get() + 64 * nranks, hbuf.get(), 64, ncclUint8, c, st), "allgather handles");
  std::vector<cudaIpcMemHandle_t> hs(nranks);
  DSG_CUDA_CHECK(cudaMemcpyAsync(hs.data(), hbuf.get(), 64 * nranks, cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  std::vector<const float*> src(nranks, nullptr);
  for (int r = 0; r < nranks && ok; ++r) {
    if (r == rank) {
      src[r] = send.get();
      continue;
    }
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = false;
      continue;
    }
    src[r] = static_cast<const float*>(p);
  }
  DevBuf<int> flag;
  flag.ensure(1);
  const int okv = ok ? 1 : 0;
  DSG_CUDA_CHECK(cudaMemcpyAsync(flag.get(), &okv, sizeof(int), cudaMemcpyHostToDevice, st));
  nc(N.AllReduce(flag.get(), flag.get(), 1, ncclInt32, ncclMin, c, st), "allreduce ipc status");
  int all_ok = 0;
  DSG_CUDA_CHECK(cudaMemcpyAsync(&all_ok, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  if (all_ok) {
    std::vector<PullPart> pp(P);
    int64_t maxc = 1;
    for (int k = 0; k < P; ++k) {
      const int r = k % nranks;
      pp[k] = PullPart{src[r] + roff[k] * kParams, cnt[k], off[k]};
      maxc = std::max(maxc, cnt[k]);
    }
    DevBuf<PullPart> dpp;
    dpp.ensure(P);
    DSG_CUDA_CHECK(cudaMemcpyAsync(dpp.get(), pp.data(), sizeof(PullPart) * P,
                                   cudaMemcpyHostToDevice, st));
    cudaEvent_t e0, e1;
    DSG_CUDA_CHECK(cudaEventCreate(&e0));
    DSG_CUDA_CHECK(cudaEventCreate(&e1));
    DSG_CUDA_CHECK(cudaEventRecord(e0, st));
    const size_t smem = sizeof(float) * kPeerRecs * kParams;
    DSG_CUDA_CHECK(cudaFuncSetAttribute(k_peer_pull, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    k_peer_pull<<<dim3((unsigned)((maxc + kPeerRecs - 1) / kPeerRecs), (unsigned)P), 256, smem,
                  st>>>(dpp.get(), merged.params.get(), merged.cap);
    count_launch();
    DSG_CUDA_CHECK(cudaEventRecord(e1, st));
    nc(N.AllReduce(flag.get(), flag.get(), 1, ncclInt32, ncclMin, c, st), "allreduce done");
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    float t = 0.f;
    DSG_CUDA_CHECK(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (wire_ms) *wire_ms = t;
  }
  for (int r = 0; r < nranks; ++r)
    if (r != rank && src[r]) cudaIpcCloseMemHandle(const_cast<float*>(src[r]));
  return all_ok != 0;
}

// Steps 1-3 above. `merged` receives the merged model (reserved inside).
// Rank r holds partitions k = j * nranks + r for j < nlocal (partition k on
// GPU k mod N, runtime.hpp:337-343 worker assignment). The survivors travel
// as packed 56 B records: one NCCL all-gather per round j, every rank's
// records padded to that round's largest count (slabs are count-balanced, so
// the padding is the ghost imbalance); one kernel per round scatters them
// into the merged planar store at their (partition, index) offsets.
int64_t merge_allgather_dev(void* comm, int nranks, int rank, const ModelDev* const* locals,
                            int nlocal, int axis, const double* cut_lo, const double* cut_hi,
                            ModelDev& merged, ScanScratch& sc, MergeScratch& ms, cudaStream_t st,
                            float* wire_ms, int64_t* max_iteration) {
  Nccl& N = nccl();
  ncclComm_t c = (ncclComm_t)comm;
  const int P = nranks * nlocal;
  // 1. local compaction of each partition into a dense [14][cnt] buffer
  std::vector<int64_t> mine(2 * nlocal);
  std::deque<DevBuf<float>>& dense = ms.dense;  // kept between calls
  if ((int)dense.size() < nlocal) dense.resize(nlocal);
  std::vector<MergeSrc> src(nlocal);
  std::vector<int64_t> lcnt(nlocal);
  for (int j = 0; j < nlocal; ++j) {
    const ModelDev& L = *locals[j];
    src[j] = {L.params.get(), L.cap, L.n, cut_lo[j], cut_hi[j]};
  }
  merge_trim_count(src.data(), nlocal, axis, ms, sc, st, lcnt.data());
  for (int j = 0; j < nlocal; ++j) {
    const int64_t cnt = lcnt[j];
    dense[j].ensure((size_t)kParams * std::max<int64_t>(cnt, 1));
    merge_trim_scatter(src[j], j, ms, dense[j].get(), std::max<int64_t>(cnt, 1), 0, st);
    mine[2 * j] = cnt;
    mine[2 * j + 1] = locals[j]->iteration;
  }
  // 2. (count, iteration) of every partition
  DevBuf<int64_t> meta;
  meta.ensure((size_t)2 * nlocal * (nranks + 1));
  int64_t* send_meta = meta.get() + (size_t)2 * nlocal * nranks;
  DSG_CUDA_CHECK(cudaMemcpyAsync(send_meta, mine.data(), sizeof(int64_t) * 2 * nlocal,
                                 cudaMemcpyHostToDevice, st));
  nc(N.AllGather(send_meta, meta.get(), (size_t)2 * nlocal, ncclInt64, c, st), "allgather counts");
  std::vector<int64_t> all((size_t)2 * nlocal * nranks);
  DSG_CUDA_CHECK(cudaMemcpyAsync(all.data(), meta.get(), sizeof(int64_t) * all.size(),
                                 cudaMemcpyDeviceToHost, st));
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  std::vector<int64_t> cnt(P), off(P);
  int64_t total = 0, it_max = 0;
  for (int k = 0; k < P; ++k) {  // partition order: merge_models (partition.hpp:117-123)
    const int r = k % nranks, j = k / nranks;
    cnt[k] = all[(size_t)r * 2 * nlocal + 2 * j];
    it_max = std::max(it_max, all[(size_t)r * 2 * nlocal + 2 * j + 1]);
    off[k] = total;
    total += cnt[k];
  }
  if (max_iteration) *max_iteration = it_max;
  // per round: counts and offsets of partitions j * N + r, r = 0..N-1
  DevBuf<int64_t> co;
  co.ensure((size_t)2 * P);
  DSG_CUDA_CHECK(cudaMemcpyAsync(co.get(), cnt.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, st));
  DSG_CUDA_CHECK(cudaMemcpyAsync(co.get() + P, off.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, st));
  merged.reserve(std::max<int64_t>(total, 1));
  merged.n = total;
  // 3a. peer-memory pull (default)
  static const std::string path = [] {
    const char* e = std::getenv("DSG_MERGE_PATH");
    return std::string(e ? e : "nccl");
  }();
  if (path == "pull" && nranks > 1 &&
      merge_pull_peers(N, c, nranks, rank, nlocal, dense, cnt, off, merged, st, wire_ms)) {
    g_merge_path = "pull";
    return total;
  }
  if (path == "push" && nranks > 1 &&
      merge_push_peers(N, c, nranks, rank, nlocal, dense, cnt, off, merged, st, wire_ms)) {
    g_merge_path = "push";
    return total;
  }
  if (path == "copy" && nranks > 1 &&
      merge_push_peers(N, c, nranks, rank, nlocal, dense, cnt, off, merged, st, wire_ms, true)) {
    g_merge_path = "copy";
    return total;
  }
  g_merge_path = "nccl";
  // 3b. pack every round, align the ranks, the rounds' all-gathers back to
  // back, then unpack. The alignment (a 4-byte all-reduce) lets the timed
  // window hold only the transfer: without it the first rank into a round
  // also waits there for the others' host-side work (count readbacks).
  // Counts padded to 64 records (3584 B, a multiple of 256 B): every rank's
  // block in the gathered buffer then starts 256 B-aligned. An unaligned
  // block (a round whose largest slab is not a multiple of 4 records) sends
  // NCCL's copy loops down a slower path: 501 -> 660+ GB/s at N = 4.
  auto pad = [](int64_t c) { return (std::max<int64_t>(c, 1) + 63) & ~int64_t(63); };
  int64_t maxc_all = 1;
  for (int k = 0; k < P; ++k) maxc_all = std::max(maxc_all, cnt[k]);
  maxc_all = pad(maxc_all);
  const size_t round_recs = (size_t)maxc_all * kParams;
  DevBuf<float> send_plain, recv_plain;
  float *sendp = nullptr, *recvp = nullptr;
  if (!exchange_buffers(comm, sizeof(float) * (round_recs * nlocal + 1),
                        sizeof(float) * round_recs * nranks * nlocal, &sendp, &recvp)) {
    sendp = send_plain.ensure(round_recs * nlocal + 1);
    recvp = recv_plain.ensure(round_recs * nranks * nlocal);
  }
  std::vector<int64_t> maxc(nlocal, 1);
  for (int j = 0; j < nlocal; ++j) {
    for (int r = 0; r < nranks; ++r) maxc[j] = std::max(maxc[j], cnt[j * nranks + r]);
    maxc[j] = pad(maxc[j]);
    const int64_t my = cnt[j * nranks + rank];
    if (my > 0) {
      k_pack_records<<<(unsigned)((my * kParams + 255) / 256), 256, 0, st>>>(
          dense[j].get(), std::max<int64_t>(my, 1), my, sendp + round_recs * j);
      count_launch();
    }
  }
  float* flag = sendp + round_recs * nlocal;
  DSG_CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(float), st));
  nc(N.AllReduce(flag, flag, 1, ncclFloat32, ncclSum, c, st), "align ranks");
  cudaEvent_t e0, e1;
  DSG_CUDA_CHECK(cudaEventCreate(&e0));
  DSG_CUDA_CHECK(cudaEventCreate(&e1));
  DSG_CUDA_CHECK(cudaEventRecord(e0, st));
  for (int j = 0; j < nlocal; ++j)
    nc(N.AllGather(sendp + round_recs * j, recvp + round_recs * nranks * j,
                   (size_t)maxc[j] * kParams, ncclFloat32, c, st),
       "allgather survivors");
  DSG_CUDA_CHECK(cudaEventRecord(e1, st));
  for (int j = 0; j < nlocal; ++j) {
    const int64_t tot_rec = (int64_t)nranks * maxc[j] * kParams;
    k_unpack_records<<<(unsigned)((tot_rec + 255) / 256), 256, 0, st>>>(
        recvp + round_recs * nranks * j, maxc[j], nranks, co.get() + (size_t)j * nranks,
        co.get() + P + (size_t)j * nranks, merged.params.get(), merged.cap);
    count_launch();
  }
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  float t = 0.f;
  DSG_CUDA_CHECK(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (wire_ms) *wire_ms = t;
  return total;
}

namespace {
__global__ void k_fill_hash(float* p, size_t n, uint32_t seed) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 0x9e3779b9u ^ seed;
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    p[i] = (float)(h & 0xffffff) * (1.f / 16777216.f);
  }
}
}  // namespace

// dsg_comm_bench_allgather: the exchange communicator's raw all-gather
// (DSG_BENCH_RANDOM=1: random-valued source instead of zeros).
double bench_allgather_dev(void* comm, int nranks, int64_t bytes, int reps, cudaStream_t st) {
  Nccl& N = nccl();
  ncclComm_t c = (ncclComm_t)comm;
  const size_t n = (size_t)std::max<int64_t>(bytes / 4, 1);
  DevBuf<float> send, recv, flag;
  send.ensure(n);
  recv.ensure(n * nranks);
  flag.ensure(1);
  DSG_CUDA_CHECK(cudaMemsetAsync(send.get(), 0, sizeof(float) * n, st));
  if (const char* e = std::getenv("DSG_BENCH_RANDOM"))
    if (e[0] == '1') k_fill_hash<<<148 * 8, 256, 0, st>>>(send.get(), n, 12345u);
  cudaEvent_t e0, e1;
  DSG_CUDA_CHECK(cudaEventCreate(&e0));
  DSG_CUDA_CHECK(cudaEventCreate(&e1));
  double tot = 0.0;
  for (int r = 0; r <= reps; ++r) {  // r = 0: warm-up
    nc(N.AllReduce(flag.get(), flag.get(), 1, ncclFloat32, ncclSum, c, st), "align ranks");
    DSG_CUDA_CHECK(cudaEventRecord(e0, st));
    nc(N.AllGather(send.get(), recv.get(), n, ncclFloat32, c, st), "allgather");
    DSG_CUDA_CHECK(cudaEventRecord(e1, st));
    DSG_CUDA_CHECK(cudaEventSynchronize(e1));
    float t = 0.f;
    DSG_CUDA_CHECK(cudaEventElapsedTime(&t, e0, e1));
    if (r > 0) tot += t;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return reps > 0 ? tot / reps : 0.0;
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
