// libdsg C ABI (include/dsg.h): host orchestration of the sm_100a kernels.
//
// Mirrors the reference entry points render (render.hpp:160), backward
// (backward.hpp:184), masked_loss (loss.hpp:39), AdamState::step
// (adam.hpp:55) and train_partition_full (trainer.hpp:140) over device-
// resident models and views. Validation order and messages follow the
// reference so the C++ wrappers can rethrow identical dsplat::Error texts.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>
#include <unistd.h>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include <nvtx3/nvToolsExt.h>

#include "../../include/dsg.h"
#include "dsg_internal.h"
#include "raster.h"

namespace dsg {

static const char* kCodeNames[] = {
    "BehindCamera", "InvalidRig", "UnknownKind", "IsovalueOutOfRange", "EmptyCloud",
    "DimensionMismatch", "TooSmall", "EmptyBand", "EmptyInterior", "MismatchedCounts", "NoViews",
    "StaleForward", "IoError", "MalformedFile", "WorkerFailure", "Timeout", "ManifestMismatch",
    "MissingBaseline", "InvalidArgument"};

void fail(int code, const std::string& msg) { throw Error{code, msg}; }

static std::atomic<int64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void throw_cuda(cudaError_t e, const char* expr, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
           cudaGetErrorString(e), file, line, expr);
  throw Error{kWorkerFailure, buf};
}

void ModelDev::reserve(int64_t c) {
  if (c <= cap) return;
  int64_t nc = std::max<int64_t>(c, 64);
  params.release(); grads.release(); m.release(); v.release(); dmean.release();
  stat_norm.release(); touch.release(); stat_count.release();
  params.ensure(kParams * nc);
  grads.ensure(kParams * nc);
  m.ensure(kParams * nc);
  v.ensure(kParams * nc);
  dmean.ensure(2 * nc);
  stat_norm.ensure(nc);
  touch.ensure(nc);
  stat_count.ensure(nc);
  cap = nc;
}

}  // namespace dsg

using namespace dsg;

struct dsg_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  Frame frame;
  DevBuf<double> stage_d;
  DevBuf<double> stage_d2;
  DevBuf<float> stage_f;
  DevBuf<uint8_t> stage_u8;
  DevBuf<double> loss_trace;
  StageTimer timer;
  bool timer_init = false;
  ModelDev spare;  // densification output storage (swapped with the model's)
  DensifyScratch dscratch;
  MergeScratch merge;  // ghost trim of merge_models / the merge exchange
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
  // end-to-end mode: next step's view is copied on its own stream into the
  // other of two device slots while this step computes
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_consumed[2] = {nullptr, nullptr};
  // pinned staging for large pageable model transfers (staged_copy)
  char* pin[2] = {nullptr, nullptr};
  // pinned per-step view slots of reference-layout host views (planar fp32 + u8)
  char* vpin[2] = {nullptr, nullptr};
  size_t vpin_bytes = 0;
  // device slots of streamed (host) views, owned by the context so creating
  // and destroying host view sets never allocates device memory
  DevBuf<float> vslot_gt;
  DevBuf<uint8_t> vslot_mask;
  cudaEvent_t pin_ev[2] = {nullptr, nullptr};
  double last_total_ms = 0.0;
  int64_t last_iters = 0;
  double last_stage_ms[StageTimer::kStages] = {};
  bool profile = false;
};

struct dsg_model_s {
  ModelDev m;
};

struct dsg_views_s {
  int32_t n = 0;
  int width = 0, height = 0;
  std::vector<dsg_camera> cams;
  DevBuf<float> gt;       // [v][3][npix] (host mode: two staging slots)
  DevBuf<uint8_t> mask;   // [v][npix] (host mode: two slots)
  bool host = false;      // views live in caller-owned pinned host memory
  std::vector<const float*> host_gt;
  std::vector<const uint8_t*> host_mask;
  // reference layout (TrainView, loss.hpp:14-26): HWC double GT + HW double
  // mask in caller memory, converted per step into pinned staging slots
  bool ref_layout = false;
  std::vector<const double*> host_gt64, host_mask64;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = std::string(kCodeNames[e.code]) + ": " + e.msg;
    cudaGetLastError();  // a reported CUDA error must not resurface in the next call
    return e.code + 1;
  } catch (const std::exception& e) {
    g_err = std::string("InvalidArgument: ") + e.what();
    cudaGetLastError();
    return kInvalidArgument + 1;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) DSG_CUDA_CHECK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// ---- host mirrors of the reference's small value types -----------------------
struct V3 {
  double x, y, z;
};
V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double norm(V3 a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
V3 unit(V3 a) {
  double n = norm(a);
  return n > 0.0 ? V3{a.x / n, a.y / n, a.z / n} : V3{0, 0, 0};
}

// Camera::validate (camera.hpp:26-36) + the constants of camera.hpp:40-62.
CamDev make_cam(const dsg_camera* c) {
  if (!c) fail(kInvalidArgument, "null camera");
  if (c->width < 8 || c->height < 8) fail(kInvalidRig, "camera resolution below 8 px");
  if (!(c->fov_y > 0.0 && c->fov_y < M_PI)) fail(kInvalidRig, "fov_y outside (0, pi)");
  if (!(c->near_plane < c->far_plane)) fail(kInvalidRig, "near must be < far");
  V3 pos{c->position[0], c->position[1], c->position[2]};
  V3 tgt{c->target[0], c->target[1], c->target[2]};
  V3 up{c->up[0], c->up[1], c->up[2]};
  V3 dir = sub(tgt, pos);
  if (norm(cross(dir, up)) <= 1e-12 * norm(dir) * norm(up))
    fail(kInvalidRig, "up parallel to view direction");
  V3 f = unit(dir);
  V3 r = unit(cross(f, up));
  V3 u = cross(r, f);
  CamDev k{};
  double R[9] = {r.x, r.y, r.z, u.x, u.y, u.z, f.x, f.y, f.z};
  std::memcpy(k.R, R, sizeof R);
  k.pos[0] = pos.x;
  k.pos[1] = pos.y;
  k.pos[2] = pos.z;
  k.f = 0.5 * c->height / std::tan(0.5 * c->fov_y);
  k.half_w = 0.5 * c->width;
  k.half_h = 0.5 * c->height;
  k.near_plane = c->near_plane;
  k.width = c->width;
  k.height = c->height;
  k.tiles_x = (c->width + kTile - 1) / kTile;
  k.tiles_y = (c->height + kTile - 1) / kTile;
  k.band_ty0 = 0;
  k.band_ty1 = k.tiles_y;
  return k;
}

// RenderConfig::validate (render.hpp:27-34).
RenderDev make_rd(const dsg_render_config* c) {
  if (!c) fail(kInvalidArgument, "null render config");
  if (c->tile_size <= 0 || (c->tile_size & (c->tile_size - 1)) != 0)
    fail(kInvalidArgument, "tile_size must be a positive power of two");
  if (!(c->alpha_cutoff > 0.0 && c->alpha_cutoff < 1.0))
    fail(kInvalidArgument, "alpha_cutoff outside (0, 1)");
  if (!(c->sigma_cutoff >= 1.0 && c->sigma_cutoff <= 6.0))
    fail(kInvalidArgument, "sigma_cutoff outside [1, 6]");
  RenderDev r{};
  r.sigma_cutoff = c->sigma_cutoff;
  r.sigma_sq = c->sigma_cutoff * c->sigma_cutoff;
  r.alpha_cutoff = c->alpha_cutoff;
  r.floor_T = c->transmittance_floor;
  for (int k = 0; k < 3; ++k) r.bg[k] = (float)c->background[k];
  for (int k = 0; k < 3; ++k) r.bg64[k] = c->background[k];
  r.sigma_sq_f = (float)r.sigma_sq;
  r.alpha_cutoff_f = (float)r.alpha_cutoff;
  r.floor_T_f = (float)r.floor_T;
  return r;
}

// ---- layout conversion kernels -------------------------------------------------
template <class A>
__global__ void k_aos_to_planar(const A* __restrict__ aos, int64_t n, int C,
                                float* __restrict__ planar, int64_t pitch) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int c = 0; c < C; ++c) planar[c * pitch + i] = (float)aos[i * C + c];
}

template <class A>
__global__ void k_planar_to_aos(const float* __restrict__ planar, int64_t pitch, int64_t n, int C,
                                A* __restrict__ aos) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int c = 0; c < C; ++c) aos[i * C + c] = (A)planar[c * pitch + i];
}

__global__ void k_mask_u8(const double* __restrict__ m, int64_t n, uint8_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = m[i] >= 0.5 ? 1 : 0;
}

__global__ void k_render_out(const float* __restrict__ rgb, const float* __restrict__ T,
                             int64_t npix, double* __restrict__ out_rgb,
                             double* __restrict__ out_alpha) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npix) return;
  for (int c = 0; c < 3; ++c) out_rgb[3 * i + c] = (double)rgb[c * npix + i];
  out_alpha[i] = 1.0 - (double)T[i];
}

__global__ void k_fill_bg(float* rgb, float* T, uint32_t* last, int32_t* nc, int64_t npix,
                          float r, float g, float b) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npix) return;
  rgb[i] = r;
  rgb[npix + i] = g;
  rgb[2 * npix + i] = b;
  T[i] = 1.f;
  last[i] = 0;
  nc[i] = 0;
}

inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

// Forward pass of one view into ctx->frame (binning + K5). An empty visible
// set leaves the background image, like render() (render.hpp:169-172).
void forward(dsg_ctx ctx, ModelDev& m, const CamDev& cam, const RenderDev& rd) {
  Frame& f = ctx->frame;
  bin_frame(f, m.params.get(), m.cap, m.n, cam, rd, ctx->stream);
  const int64_t npix = (int64_t)cam.width * cam.height;
  if (f.n_visible == 0 || f.n_dup == 0) {
    f.width = cam.width;
    f.height = cam.height;
    f.rgb.ensure(3 * npix);
    f.T.ensure(npix);
    f.last.ensure(npix);
    f.ncontrib.ensure(npix);
    k_fill_bg<<<nblk(npix), 256, 0, ctx->stream>>>(f.rgb.get(), f.T.get(), f.last.get(),
                                                   f.ncontrib.get(), npix, rd.bg[0], rd.bg[1],
                                                   rd.bg[2]);
                                                   count_launch();
    return;
  }
  blend_forward(f, m.params.get(), m.cap, cam, rd, ctx->stream);
}

// K6 + K7 on the current frame (forward and f.dL must be in place).
void backward_dev(dsg_ctx ctx, ModelDev& m, const CamDev& cam, const RenderDev& rd) {
  Frame& f = ctx->frame;
  blend_backward(f, m.params.get(), m.cap, cam, rd, ctx->stream);
  ChainArgs a;
  a.params = m.params.get();
  a.pitch = m.cap;
  a.n = m.n;
  a.cam = cam;
  a.tcount = f.tcount.get();
  a.dup_base = f.dup_base.get();
  a.partials = f.partials.get();
  a.n_dup = f.n_dup;
  a.tmask = f.tmask.get();
  a.grads = m.grads.get();
  a.dmean = m.dmean.get();
  a.touch = m.touch.get();
  if (f.n_visible == 0 || f.n_dup == 0) {
    // nothing visible: all gradients are exactly zero (backward.hpp:195)
    DSG_CUDA_CHECK(cudaMemsetAsync(m.grads.get(), 0, sizeof(float) * kParams * m.cap, ctx->stream));
    DSG_CUDA_CHECK(cudaMemsetAsync(m.dmean.get(), 0, sizeof(float) * 2 * m.cap, ctx->stream));
    DSG_CUDA_CHECK(cudaMemsetAsync(m.touch.get(), 0, sizeof(int32_t) * m.cap, ctx->stream));
    return;
  }
  chain_3d(a, ctx->stream);
}

AdamArgs make_adam(ModelDev& m, const double* rates, const dsg_adam_config& ac, int64_t step,
                   bool stats) {
  AdamArgs a;
  a.params = m.params.get();
  a.grads = m.grads.get();
  a.m = m.m.get();
  a.v = m.v.get();
  a.dmean = m.dmean.get();
  a.touch = m.touch.get();
  a.stat_norm = m.stat_norm.get();
  a.stat_count = m.stat_count.get();
  a.pitch = m.cap;
  a.n = m.n;
  for (int k = 0; k < 5; ++k) a.lr[k] = (float)rates[k];
  a.b1 = (float)ac.beta1;
  a.b2 = (float)ac.beta2;
  a.omb1 = (float)(1.0 - ac.beta1);
  a.omb2 = (float)(1.0 - ac.beta2);
  double bc1 = 1.0 - std::pow(ac.beta1, (double)step);
  double bc2 = 1.0 - std::pow(ac.beta2, (double)step);
  a.inv_bc1 = (float)(1.0 / bc1);
  a.inv_bc2 = (float)(1.0 / bc2);
  a.eps = (float)ac.epsilon;
  a.ls_lo = (float)std::log(1e-7);
  a.ls_hi = (float)std::log(1e3);
  a.accumulate_stats = stats ? 1 : 0;
  return a;
}

void reset_optimizer(dsg_ctx ctx, ModelDev& m) {
  cudaStream_t st = ctx->stream;
  DSG_CUDA_CHECK(cudaMemsetAsync(m.m.get(), 0, sizeof(float) * kParams * m.cap, st));
  DSG_CUDA_CHECK(cudaMemsetAsync(m.v.get(), 0, sizeof(float) * kParams * m.cap, st));
  DSG_CUDA_CHECK(cudaMemsetAsync(m.stat_norm.get(), 0, sizeof(double) * m.cap, st));
  DSG_CUDA_CHECK(cudaMemsetAsync(m.stat_count.get(), 0, sizeof(int32_t) * m.cap, st));
  m.adam_step = 0;
}

// splitmix64 stream of rng.hpp:8-64 (view order shuffle, trainer.hpp:160-163).
struct Rng {
  uint64_t s;
  static uint64_t mix(uint64_t& st) {
    st += 0x9e3779b97f4a7c15ULL;
    uint64_t z = st;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  explicit Rng(uint64_t seed) : s(seed ^ 0x853c49e6748fea9bULL) {
    mix(s);
    mix(s);
  }
  uint64_t below(uint64_t n) { return n > 0 ? mix(s) % n : 0; }
};

void validate_train(const dsg_train_config* c) {  // trainer.hpp:31-38
  if (c->lr_mu <= 0 || c->lr_scale <= 0 || c->lr_rot <= 0 || c->lr_opacity <= 0 || c->lr_color <= 0)
    fail(kInvalidArgument, "learning rates must be positive");
  if (c->loss_lambda < 0.0 || c->loss_lambda > 1.0)
    fail(kInvalidArgument, "loss_lambda outside [0, 1]");
  if (c->iterations < 0) fail(kInvalidArgument, "iterations must be >= 0");
}

}  // namespace

extern "C" {

const char* dsg_last_error(void) { return g_err.c_str(); }
int32_t dsg_abi_version(void) { return DSG_ABI_VERSION; }

int dsg_ctx_create(int32_t device, dsg_ctx* out) {
  return guarded([&] {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) fail(kInvalidArgument, "no CUDA device available");
    if (device < 0 || device >= count) fail(kInvalidArgument, "device index out of range");
    cudaDeviceProp prop;
    DSG_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) fail(kInvalidArgument, "libdsg is built for sm_100a (B200) only");
    auto* c = new dsg_ctx_s();
    c->device = device;
    DeviceGuard g(device);
    DSG_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    // the two 32 MiB pinned staging chunks of large model transfers are part
    // of the context (pinning them costs tens of ms on a cold host)
    for (int k = 0; k < 2; ++k) {
      DSG_CUDA_CHECK(cudaMallocHost(&c->pin[k], size_t(32) << 20));
      DSG_CUDA_CHECK(cudaEventCreateWithFlags(&c->pin_ev[k], cudaEventDisableTiming));
    }
    *out = c;
  });
}

int dsg_ctx_destroy(dsg_ctx ctx) {
  return guarded([&] {
    if (!ctx) return;
    DeviceGuard g(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->timer_init) {
      for (int k = 0; k <= StageTimer::kStages; ++k) cudaEventDestroy(ctx->timer.ev[k]);
      cudaEventDestroy(ctx->ev_begin);
      cudaEventDestroy(ctx->ev_end);
    }
    for (int k = 0; k < 2; ++k) {
      if (ctx->ev_copied[k]) cudaEventDestroy(ctx->ev_copied[k]);
      if (ctx->ev_consumed[k]) cudaEventDestroy(ctx->ev_consumed[k]);
    }
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    for (int k = 0; k < 2; ++k) {
      if (ctx->pin[k]) cudaFreeHost(ctx->pin[k]);
      if (ctx->vpin[k]) cudaFreeHost(ctx->vpin[k]);
      if (ctx->pin_ev[k]) cudaEventDestroy(ctx->pin_ev[k]);
    }
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int dsg_ctx_synchronize(dsg_ctx ctx) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  });
}

int dsg_model_create(dsg_ctx ctx, dsg_model* out) {
  return guarded([&] {
    (void)ctx;
    *out = new dsg_model_s();
  });
}

int dsg_model_destroy(dsg_model model) {
  return guarded([&] { delete model; });
}

namespace {

// Host worker pool for the staged copies: created once, reused by every
// chunk (spawning 16 threads per 32 MiB chunk cost ~0.3 ms a chunk).
class HostPool {
 public:
  static HostPool& get() {
    static HostPool p;
    return p;
  }
  int size() const { return (int)workers_.size() + 1; }
  // fn(i) for i in [0, n) on the workers and the caller; returns when all are done
  void run(int n, const std::function<void(int)>& fn) {
    if (getpid() != pid_) {  // a forked child has no workers: run inline
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    std::lock_guard<std::mutex> one(run_mu_);  // one job at a time
    std::unique_lock<std::mutex> lk(mu_);
    fn_ = &fn;
    n_ = n;
    next_ = 1;
    pending_ = n - 1;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    fn(0);
    lk.lock();
    while (true) {  // the caller helps with items no worker has claimed yet
      if (next_ >= n_) break;
      const int i = next_++;
      lk.unlock();
      fn(i);
      lk.lock();
      --pending_;
    }
    done_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  HostPool() : pid_(getpid()) {
    // ranks of one node share its cores (torchrun sets LOCAL_WORLD_SIZE)
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    if (const char* lw = std::getenv("LOCAL_WORLD_SIZE")) {
      const int k = std::atoi(lw);
      if (k > 1) hw = std::max(1u, hw / (unsigned)k);
    }
    for (unsigned k = 1; k < std::min(hw, 16u); ++k)
      workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    if (getpid() != pid_) {  // forked child: the workers (and mu_'s owner) are the parent's
      for (auto& t : workers_) t.detach();
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void loop() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    while (true) {
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      while (fn_ && next_ < n_) {
        const int i = next_++;
        const std::function<void(int)>* fn = fn_;
        lk.unlock();
        (*fn)(i);
        lk.lock();
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  const pid_t pid_;
  std::vector<std::thread> workers_;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0, next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Copy between a large pageable host buffer and device memory: 32 MiB chunks
// through two pinned staging buffers, the DMA of one chunk overlapping a
// multi-threaded host memcpy of the other (a single pageable cudaMemcpy is
// bound by the driver's one-thread staging copy and first-touch faults).
void par_memcpy(char* dst, const char* src, size_t n) {
  const size_t kMinPerThread = 1 << 20;
  HostPool& pool = HostPool::get();
  const size_t nt = std::min<size_t>((size_t)pool.size(), (n + kMinPerThread - 1) / kMinPerThread);
  if (nt <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  const size_t per = ((n + nt - 1) / nt + 4095) & ~size_t(4095);
  pool.run((int)((n + per - 1) / per), [=](int k) {
    const size_t o = (size_t)k * per;
    std::memcpy(dst + o, src + o, std::min(per, n - o));
  });
}

// Model parameters cross the bus as fp32 (what the device stores): the host
// side converts double <-> float in parallel while the pinned chunks are in
// flight, halving the bytes a pageable double copy would move. The rounding
// is the device's own cast (round to nearest), so results are unchanged.
}  // namespace
}  // extern "C"
namespace {
// Streaming (non-temporal) stores: the converted data is not read again by
// this thread, and skipping the read-for-ownership of the destination cuts
// host DRAM traffic by a third. Same rounding as the scalar cast (MXCSR
// round-to-nearest, cvtpd2ps / cvtps2pd).
inline void convert_span(double* dst, const float* src, size_t n) {
  size_t i = 0;
#if defined(__SSE2__)
  for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 15); ++i) dst[i] = (double)src[i];
  for (; i + 2 <= n; i += 2) {
    const __m128 f = _mm_castpd_ps(_mm_load_sd(reinterpret_cast<const double*>(src + i)));
    _mm_stream_pd(dst + i, _mm_cvtps_pd(f));
  }
  _mm_sfence();
#endif
  for (; i < n; ++i) dst[i] = (double)src[i];
}
inline void convert_span(float* dst, const double* src, size_t n) {
  size_t i = 0;
#if defined(__SSE2__)
  for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 15); ++i) dst[i] = (float)src[i];
  for (; i + 4 <= n; i += 4) {
    const __m128 lo = _mm_cvtpd_ps(_mm_loadu_pd(src + i));
    const __m128 hi = _mm_cvtpd_ps(_mm_loadu_pd(src + i + 2));
    _mm_stream_ps(dst + i, _mm_movelh_ps(lo, hi));
  }
  _mm_sfence();
#endif
  for (; i < n; ++i) dst[i] = (float)src[i];
}

template <class H, class D>
void par_convert(D* dst, const H* src, size_t n) {
  const size_t kMin = size_t(1) << 18;
  HostPool& pool = HostPool::get();
  const size_t nt = std::min<size_t>((size_t)pool.size(), (n + kMin - 1) / kMin);
  if (nt <= 1) {
    convert_span(dst, src, n);
    return;
  }
  const size_t per = (((n + nt - 1) / nt) + 15) & ~size_t(15);
  pool.run((int)((n + per - 1) / per), [=](int k) {
    const size_t o = (size_t)k * per;
    convert_span(dst + o, src + o, std::min(per, n - o));
  });
}
}  // namespace
extern "C" {
namespace {

void staged_params(dsg_ctx ctx, double* host, float* dev, size_t count, bool to_host) {
  constexpr size_t kChunk = size_t(8) << 20;  // floats per pinned chunk (32 MiB)
  cudaStream_t st = ctx->stream;
  for (int k = 0; k < 2; ++k) {
    if (!ctx->pin[k]) DSG_CUDA_CHECK(cudaMallocHost(&ctx->pin[k], size_t(32) << 20));
    if (!ctx->pin_ev[k]) DSG_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->pin_ev[k], cudaEventDisableTiming));
  }
  float* pin[2] = {reinterpret_cast<float*>(ctx->pin[0]), reinterpret_cast<float*>(ctx->pin[1])};
  const size_t nch = (count + kChunk - 1) / kChunk;
  auto len = [&](size_t k) { return std::min(kChunk, count - k * kChunk); };
  if (to_host) {
    DSG_CUDA_CHECK(cudaMemcpyAsync(pin[0], dev, sizeof(float) * len(0), cudaMemcpyDeviceToHost, st));
    DSG_CUDA_CHECK(cudaEventRecord(ctx->pin_ev[0], st));
    for (size_t k = 0; k < nch; ++k) {
      if (k + 1 < nch) {
        const int b = (int)((k + 1) & 1);
        DSG_CUDA_CHECK(cudaMemcpyAsync(pin[b], dev + (k + 1) * kChunk, sizeof(float) * len(k + 1),
                                       cudaMemcpyDeviceToHost, st));
        DSG_CUDA_CHECK(cudaEventRecord(ctx->pin_ev[b], st));
      }
      DSG_CUDA_CHECK(cudaEventSynchronize(ctx->pin_ev[k & 1]));
      par_convert<float, double>(host + k * kChunk, pin[k & 1], len(k));
    }
  } else {
    for (size_t k = 0; k < nch; ++k) {
      const int b = (int)(k & 1);
      if (k >= 2) DSG_CUDA_CHECK(cudaEventSynchronize(ctx->pin_ev[b]));
      par_convert<double, float>(pin[b], host + k * kChunk, len(k));
      DSG_CUDA_CHECK(cudaMemcpyAsync(dev + k * kChunk, pin[b], sizeof(float) * len(k),
                                     cudaMemcpyHostToDevice, st));
      DSG_CUDA_CHECK(cudaEventRecord(ctx->pin_ev[b], st));
    }
  }
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
}

void staged_copy(dsg_ctx ctx, char* host, char* dev, size_t bytes, bool to_host) {
  constexpr size_t kChunk = size_t(32) << 20;
  cudaStream_t st = ctx->stream;
  if (bytes < (size_t(8) << 20)) {
    DSG_CUDA_CHECK(cudaMemcpyAsync(to_host ? (void*)host : (void*)dev, to_host ? (void*)dev : (void*)host,
                                   bytes, to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, st));
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    return;
  }
  for (int k = 0; k < 2; ++k) {
    if (!ctx->pin[k]) DSG_CUDA_CHECK(cudaMallocHost(&ctx->pin[k], kChunk));
    if (!ctx->pin_ev[k]) DSG_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->pin_ev[k], cudaEventDisableTiming));
  }
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  auto len = [&](size_t k) { return std::min(kChunk, bytes - k * kChunk); };
  if (to_host) {
    DSG_CUDA_CHECK(cudaMemcpyAsync(ctx->pin[0], dev, len(0), cudaMemcpyDeviceToHost, st));
    DSG_CUDA_CHECK(cudaEventRecord(ctx->pin_ev[0], st));
    for (size_t k = 0; k < nch; ++k) {
      if (k + 1 < nch) {  // its buffer's previous chunk (k-1) was drained last iteration
        const int b = (int)((k + 1) & 1);
        DSG_CUDA_CHECK(cudaMemcpyAsync(ctx->pin[b], dev + (k + 1) * kChunk, len(k + 1),
                                       cudaMemcpyDeviceToHost, st));
        DSG_CUDA_CHECK(cudaEventRecord(ctx->pin_ev[b], st));
      }
      DSG_CUDA_CHECK(cudaEventSynchronize(ctx->pin_ev[k & 1]));
      par_memcpy(host + k * kChunk, ctx->pin[k & 1], len(k));
    }
  } else {
    for (size_t k = 0; k < nch; ++k) {
      const int b = (int)(k & 1);
      if (k >= 2) DSG_CUDA_CHECK(cudaEventSynchronize(ctx->pin_ev[b]));  // buffer's DMA done
      par_memcpy(ctx->pin[b], host + k * kChunk, len(k));
      DSG_CUDA_CHECK(cudaMemcpyAsync(dev + k * kChunk, ctx->pin[b], len(k), cudaMemcpyHostToDevice, st));
      DSG_CUDA_CHECK(cudaEventRecord(ctx->pin_ev[b], st));
    }
  }
  DSG_CUDA_CHECK(cudaStreamSynchronize(st));
}

}  // namespace

int dsg_model_upload(dsg_ctx ctx, dsg_model model, const double* params, int64_t n,
                     int64_t iteration, int32_t origin_partition) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    if (n < 0) fail(kInvalidArgument, "negative model size");
    ModelDev& m = model->m;
    m.reserve(std::max<int64_t>(n, 1));
    m.n = n;
    m.iteration = iteration;
    m.origin_partition = origin_partition;
    if (n > 0) {
      float* st = ctx->stage_f.ensure(kParams * n);
      staged_params(ctx, const_cast<double*>(params), st, (size_t)kParams * n, false);
      k_aos_to_planar<<<nblk(n), 256, 0, ctx->stream>>>(st, n, kParams, m.params.get(), m.cap);
      count_launch();
    }
    reset_optimizer(ctx, m);
    DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  });
}

int dsg_model_set_params(dsg_ctx ctx, dsg_model model, const double* params, int64_t n,
                         int64_t iteration) {
  return guarded([&] {
    ModelDev& m = model->m;
    if (n != m.n) fail(kMismatchedCounts, "model size differs from the device model");
    DeviceGuard g(ctx->device);
    m.iteration = iteration;
    if (n > 0) {
      float* st = ctx->stage_f.ensure(kParams * n);
      staged_params(ctx, const_cast<double*>(params), st, (size_t)kParams * n, false);
      k_aos_to_planar<<<nblk(n), 256, 0, ctx->stream>>>(st, n, kParams, m.params.get(), m.cap);
      count_launch();
    }
    DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  });
}

int dsg_model_download(dsg_ctx ctx, dsg_model model, double* params, int64_t capacity,
                       int64_t* n, int64_t* iteration, int32_t* origin_partition) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    ModelDev& m = model->m;
    if (n) *n = m.n;
    if (iteration) *iteration = m.iteration;
    if (origin_partition) *origin_partition = m.origin_partition;
    if (!params || m.n == 0) return;
    if (capacity < m.n) fail(kInvalidArgument, "output capacity too small");
    float* st = ctx->stage_f.ensure(kParams * m.n);
    k_planar_to_aos<<<nblk(m.n), 256, 0, ctx->stream>>>(m.params.get(), m.cap, m.n, kParams, st);
    count_launch();
    staged_params(ctx, params, st, (size_t)kParams * m.n, true);
  });
}

int dsg_model_save_ply(dsg_ctx ctx, dsg_model model, const char* path) {
  return guarded([&] {  // write_splat_ply (ply_io.hpp:89-119)
    if (!path) fail(kInvalidArgument, "null path");
    DeviceGuard g(ctx->device);
    ModelDev& m = model->m;
    const int64_t it = m.iteration;
    const int32_t op = m.origin_partition;
    const std::string head = ply_header(splat_ply_props(), kParams, m.n, &it, &op);
    std::vector<char> body((size_t)m.n * kParams * sizeof(double));
    if (m.n > 0) {
      double* d = ctx->stage_d.ensure(kParams * m.n);
      splat_ply_payload_dev(m.params.get(), m.cap, m.n, d, ctx->stream);
      staged_copy(ctx, body.data(), reinterpret_cast<char*>(d), body.size(), true);
    }
    write_file_atomic(path, head, body.data(), body.size());
  });
}

int dsg_model_load_ply(dsg_ctx ctx, dsg_model model, const char* path) {
  return guarded([&] {  // read_splat_ply (ply_io.hpp:121-158); resets the optimizer like upload
    if (!path) fail(kInvalidArgument, "null path");
    const std::string bytes = read_file(path);
    const PlyInfo h = parse_ply(bytes, splat_ply_props(), kParams, "splat");
    DeviceGuard g(ctx->device);
    ModelDev& m = model->m;
    m.reserve(std::max<int64_t>(h.vertex_count, 1));
    m.n = h.vertex_count;
    m.iteration = h.iteration;
    m.origin_partition = h.origin;
    if (m.n > 0) {
      double* d = ctx->stage_d.ensure(kParams * m.n);
      staged_copy(ctx, const_cast<char*>(bytes.data()) + h.payload_offset,
                  reinterpret_cast<char*>(d), (size_t)m.n * kParams * sizeof(double), false);
      splat_ply_scatter_dev(d, m.n, m.params.get(), m.cap, ctx->stream);
    }
    reset_optimizer(ctx, m);
    DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  });
}

int dsg_cloud_save_ply(const char* path, const double* positions, const double* normals,
                       const double* colors, int64_t n) {
  return guarded([&] {  // write_cloud_ply (ply_io.hpp:170-191)
    if (!path || n < 0) fail(kInvalidArgument, "bad cloud arguments");
    const std::string head = ply_header(cloud_ply_props(), 9, n, nullptr, nullptr);
    std::vector<double> body(9 * (size_t)n);
    for (int64_t i = 0; i < n; ++i)
      for (int c = 0; c < 3; ++c) {
        body[9 * i + c] = positions[3 * i + c];
        body[9 * i + 3 + c] = normals ? normals[3 * i + c] : 0.0;
        body[9 * i + 6 + c] = colors ? colors[3 * i + c] : 0.0;
      }
    write_file_atomic(path, head, reinterpret_cast<const char*>(body.data()),
                      body.size() * sizeof(double));
  });
}

int dsg_cloud_load_ply(const char* path, double* positions, double* normals, double* colors,
                       int64_t capacity, int64_t* n) {
  return guarded([&] {  // read_cloud_ply (ply_io.hpp:193-221)
    if (!path || !n) fail(kInvalidArgument, "bad cloud arguments");
    const std::string bytes = read_file(path);
    const PlyInfo h = parse_ply(bytes, cloud_ply_props(), 9, "cloud");
    *n = h.vertex_count;
    if (!positions) return;  // size query
    if (capacity < h.vertex_count) fail(kInvalidArgument, "output capacity too small");
    const double* src = reinterpret_cast<const double*>(bytes.data() + h.payload_offset);
    std::vector<double> row(9);
    for (int64_t i = 0; i < h.vertex_count; ++i) {
      std::memcpy(row.data(), src + 9 * i, sizeof(double) * 9);  // payload may be unaligned
      for (int c = 0; c < 3; ++c) {
        positions[3 * i + c] = row[c];
        if (normals) normals[3 * i + c] = row[3 + c];
        if (colors) colors[3 * i + c] = row[6 + c];
      }
    }
  });
}

int dsg_model_info(dsg_model model, int64_t* n, int64_t* iteration, int64_t* adam_step) {
  return guarded([&] {
    if (n) *n = model->m.n;
    if (iteration) *iteration = model->m.iteration;
    if (adam_step) *adam_step = model->m.adam_step;
  });
}

int dsg_model_adam_state(dsg_ctx ctx, dsg_model model, double* mo, double* vo, int64_t* step) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    ModelDev& m = model->m;
    if (step) *step = m.adam_step;
    if (m.n == 0) return;
    double* st = ctx->stage_d.ensure(kParams * m.n);
    for (int w = 0; w < 2; ++w) {
      double* out = w == 0 ? mo : vo;
      if (!out) continue;
      k_planar_to_aos<<<nblk(m.n), 256, 0, ctx->stream>>>(w == 0 ? m.m.get() : m.v.get(), m.cap,
                                                          m.n, kParams, st);
                                                          count_launch();
      DSG_CUDA_CHECK(cudaMemcpyAsync(out, st, sizeof(double) * kParams * m.n,
                                     cudaMemcpyDeviceToHost, ctx->stream));
      DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    }
  });
}

int dsg_model_adam_restore(dsg_ctx ctx, dsg_model model, const double* mo, const double* vo,
                           int64_t n, int64_t step) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    ModelDev& m = model->m;
    if (n != m.n) fail(kMismatchedCounts, "moment count differs from the device model");
    if (step < 0) fail(kInvalidArgument, "negative Adam step");
    cudaStream_t st = ctx->stream;
    if (n > 0) {
      double* d = ctx->stage_d.ensure(kParams * n);
      for (int k = 0; k < 2; ++k) {
        const double* src = k == 0 ? mo : vo;
        float* dst = k == 0 ? m.m.get() : m.v.get();
        if (src) {
          DSG_CUDA_CHECK(cudaMemcpyAsync(d, src, sizeof(double) * kParams * n,
                                         cudaMemcpyHostToDevice, st));
          k_aos_to_planar<<<nblk(n), 256, 0, st>>>(d, n, kParams, dst, m.cap);
          count_launch();
        } else {
          DSG_CUDA_CHECK(cudaMemsetAsync(dst, 0, sizeof(float) * kParams * m.cap, st));
        }
      }
    }
    m.adam_step = step;
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

int dsg_render(dsg_ctx ctx, dsg_model model, const dsg_camera* cam_in,
               const dsg_render_config* cfg, double* rgb, double* alpha, int32_t* n_contrib,
               int32_t* splat_order, int64_t* n_order, int64_t* model_iteration) {
  return guarded([&] {
    RenderDev rd = make_rd(cfg);   // cfg.validate() first, like render.hpp:161
    CamDev cam = make_cam(cam_in);
    DeviceGuard g(ctx->device);
    ModelDev& m = model->m;
    forward(ctx, m, cam, rd);
    Frame& f = ctx->frame;
    const int64_t npix = (int64_t)cam.width * cam.height;
    cudaStream_t st = ctx->stream;
    if (rgb || alpha) {
      double* d = ctx->stage_d.ensure(4 * npix);
      k_render_out<<<nblk(npix), 256, 0, st>>>(f.rgb.get(), f.T.get(), npix, d, d + 3 * npix);
      count_launch();
      if (rgb)
        DSG_CUDA_CHECK(cudaMemcpyAsync(rgb, d, sizeof(double) * 3 * npix, cudaMemcpyDeviceToHost, st));
      if (alpha)
        DSG_CUDA_CHECK(cudaMemcpyAsync(alpha, d + 3 * npix, sizeof(double) * npix,
                                       cudaMemcpyDeviceToHost, st));
    }
    if (n_contrib)
      DSG_CUDA_CHECK(cudaMemcpyAsync(n_contrib, f.ncontrib.get(), sizeof(int32_t) * npix,
                                     cudaMemcpyDeviceToHost, st));
    if (n_order) *n_order = f.n_visible;
    if (splat_order && f.n_visible > 0)
      DSG_CUDA_CHECK(cudaMemcpyAsync(splat_order, f.sorted_idx, sizeof(int32_t) * f.n_visible,
                                     cudaMemcpyDeviceToHost, st));
    if (model_iteration) *model_iteration = m.iteration;
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

int dsg_bin(dsg_ctx ctx, dsg_model model, const dsg_camera* cam_in, const dsg_render_config* cfg,
            int32_t* tile_count, int32_t* entries, int64_t capacity, int64_t* n_entries) {
  return guarded([&] {
    RenderDev rd = make_rd(cfg);
    CamDev cam = make_cam(cam_in);
    DeviceGuard g(ctx->device);
    Frame& f = ctx->frame;
    bin_frame(f, model->m.params.get(), model->m.cap, model->m.n, cam, rd, ctx->stream);
    *n_entries = f.n_dup;
    std::vector<uint2> ranges(f.tiles);
    DSG_CUDA_CHECK(cudaMemcpyAsync(ranges.data(), f.ranges.get(), sizeof(uint2) * f.tiles,
                                   cudaMemcpyDeviceToHost, ctx->stream));
    if (f.n_dup > capacity) fail(kInvalidArgument, "entry capacity too small");
    if (f.n_dup > 0)
      DSG_CUDA_CHECK(cudaMemcpyAsync(entries, f.sorted_val, sizeof(int32_t) * f.n_dup,
                                     cudaMemcpyDeviceToHost, ctx->stream));
    DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    for (int64_t t = 0; t < f.tiles; ++t) tile_count[t] = (int32_t)(ranges[t].y - ranges[t].x);
  });
}

int dsg_masked_loss(dsg_ctx ctx, const double* rendered, const double* ground_truth,
                    const double* mask, int32_t width, int32_t height, double loss_lambda,
                    double* loss, double* dL_dpixels) {
  return guarded([&] {
    if (width <= 0 || height <= 0) fail(kDimensionMismatch, "image dimensions differ");
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    Frame& f = ctx->frame;
    const int64_t npix = (int64_t)width * height;
    double* d = ctx->stage_d.ensure(7 * npix);
    DSG_CUDA_CHECK(cudaMemcpyAsync(d, rendered, sizeof(double) * 3 * npix, cudaMemcpyHostToDevice, st));
    DSG_CUDA_CHECK(cudaMemcpyAsync(d + 3 * npix, ground_truth, sizeof(double) * 3 * npix,
                                   cudaMemcpyHostToDevice, st));
    DSG_CUDA_CHECK(cudaMemcpyAsync(d + 6 * npix, mask, sizeof(double) * npix, cudaMemcpyHostToDevice, st));
    f.rgb.ensure(3 * npix);
    float* gt = ctx->stage_f.ensure(3 * npix);
    uint8_t* m8 = ctx->stage_u8.ensure(npix);
    k_aos_to_planar<<<nblk(npix), 256, 0, st>>>(d, npix, 3, f.rgb.get(), npix);
    count_launch();
    k_aos_to_planar<<<nblk(npix), 256, 0, st>>>(d + 3 * npix, npix, 3, gt, npix);
    count_launch();
    k_mask_u8<<<nblk(npix), 256, 0, st>>>(d + 6 * npix, npix, m8);
    count_launch();
    masked_loss_dev(f, gt, m8, width, height, loss_lambda, st);
    k_planar_to_aos<<<nblk(npix), 256, 0, st>>>(f.dL.get(), npix, npix, 3, d);
    count_launch();
    DSG_CUDA_CHECK(cudaMemcpyAsync(dL_dpixels, d, sizeof(double) * 3 * npix, cudaMemcpyDeviceToHost, st));
    DSG_CUDA_CHECK(cudaMemcpyAsync(loss, f.loss_out.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

int dsg_backward(dsg_ctx ctx, dsg_model model, const dsg_camera* cam_in,
                 const dsg_render_config* cfg, int64_t output_iteration,
                 const double* dL_dpixels, int32_t shards, double* grads, double* d_mean2d,
                 int32_t* touch_count) {
  return guarded([&] {
    ModelDev& m = model->m;
    // checks in the order of backward.hpp:187-192
    if (output_iteration != m.iteration)
      fail(kStaleForward, "render output is from a different model iteration");
    if (!cam_in || !dL_dpixels) fail(kDimensionMismatch, "dL_dpixels must be RGB at camera resolution");
    if (shards < 1) fail(kInvalidArgument, "shards must be >= 1");
    RenderDev rd = make_rd(cfg);
    CamDev cam = make_cam(cam_in);
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    Frame& f = ctx->frame;
    const int64_t npix = (int64_t)cam.width * cam.height;
    forward(ctx, m, cam, rd);
    double* d = ctx->stage_d.ensure(std::max<int64_t>(3 * npix, kParams * std::max<int64_t>(m.n, 1)));
    DSG_CUDA_CHECK(cudaMemcpyAsync(d, dL_dpixels, sizeof(double) * 3 * npix, cudaMemcpyHostToDevice, st));
    f.dL.ensure(3 * npix);
    k_aos_to_planar<<<nblk(npix), 256, 0, st>>>(d, npix, 3, f.dL.get(), npix);
    count_launch();
    backward_dev(ctx, m, cam, rd);
    if (m.n > 0) {
      if (grads) {
        k_planar_to_aos<<<nblk(m.n), 256, 0, st>>>(m.grads.get(), m.cap, m.n, kParams, d);
        count_launch();
        DSG_CUDA_CHECK(cudaMemcpyAsync(grads, d, sizeof(double) * kParams * m.n, cudaMemcpyDeviceToHost, st));
        DSG_CUDA_CHECK(cudaStreamSynchronize(st));
      }
      if (d_mean2d) {
        k_planar_to_aos<<<nblk(m.n), 256, 0, st>>>(m.dmean.get(), m.cap, m.n, 2, d);
        count_launch();
        DSG_CUDA_CHECK(cudaMemcpyAsync(d_mean2d, d, sizeof(double) * 2 * m.n, cudaMemcpyDeviceToHost, st));
        DSG_CUDA_CHECK(cudaStreamSynchronize(st));
      }
      if (touch_count)
        DSG_CUDA_CHECK(cudaMemcpyAsync(touch_count, m.touch.get(), sizeof(int32_t) * m.n,
                                       cudaMemcpyDeviceToHost, st));
    }
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

int dsg_adam_step(dsg_ctx ctx, dsg_model model, const double* grads, const dsg_group_rates* rates,
                  const dsg_adam_config* adam) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    ModelDev& m = model->m;
    cudaStream_t st = ctx->stream;
    m.adam_step += 1;
    if (m.n == 0) return;
    double* d = ctx->stage_d.ensure(kParams * m.n);
    DSG_CUDA_CHECK(cudaMemcpyAsync(d, grads, sizeof(double) * kParams * m.n, cudaMemcpyHostToDevice, st));
    k_aos_to_planar<<<nblk(m.n), 256, 0, st>>>(d, m.n, kParams, m.grads.get(), m.cap);
    count_launch();
    double r[5] = {rates->mu, rates->log_scale, rates->rot, rates->opacity, rates->color};
    adam_update(make_adam(m, r, *adam, m.adam_step, false), st);
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

int dsg_views_create(dsg_ctx ctx, const dsg_camera* cams, const double* ground_truth,
                     const double* masks, int32_t n_views, dsg_views* out) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    auto* v = new dsg_views_s();
    try {
      v->n = n_views;
      if (n_views > 0) {
        v->width = cams[0].width;
        v->height = cams[0].height;
        for (int32_t i = 0; i < n_views; ++i) {
          make_cam(&cams[i]);
          if (cams[i].width != v->width || cams[i].height != v->height)
            fail(kDimensionMismatch, "all views must share one resolution");
          v->cams.push_back(cams[i]);
        }
        const int64_t npix = (int64_t)v->width * v->height;
        v->gt.ensure(3 * npix * n_views);
        v->mask.ensure(npix * n_views);
        double* d = ctx->stage_d.ensure(4 * npix);
        for (int32_t i = 0; i < n_views; ++i) {
          DSG_CUDA_CHECK(cudaMemcpyAsync(d, ground_truth + 3 * npix * i, sizeof(double) * 3 * npix,
                                         cudaMemcpyHostToDevice, ctx->stream));
          DSG_CUDA_CHECK(cudaMemcpyAsync(d + 3 * npix, masks + npix * i, sizeof(double) * npix,
                                         cudaMemcpyHostToDevice, ctx->stream));
          k_aos_to_planar<<<nblk(npix), 256, 0, ctx->stream>>>(d, npix, 3, v->gt.get() + 3 * npix * i, npix);
          count_launch();
          k_mask_u8<<<nblk(npix), 256, 0, ctx->stream>>>(d + 3 * npix, npix, v->mask.get() + npix * i);
          count_launch();
        }
        DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
      }
    } catch (...) {
      delete v;
      throw;
    }
    *out = v;
  });
}

int dsg_views_destroy(dsg_views views) {
  return guarded([&] { delete views; });
}

int dsg_views_download(dsg_ctx ctx, dsg_views views, int32_t i, double* ground_truth,
                       double* mask) {
  return guarded([&] {
    if (views->host) fail(kInvalidArgument, "host views are already in host memory");
    if (i < 0 || i >= views->n) fail(kInvalidArgument, "view index out of range");
    DeviceGuard g(ctx->device);
    const int64_t npix = (int64_t)views->width * views->height;
    double* d = ctx->stage_d.ensure(3 * npix);
    if (ground_truth) {
      k_planar_to_aos<<<nblk(npix), 256, 0, ctx->stream>>>(views->gt.get() + 3 * npix * i, npix,
                                                           npix, 3, d);
                                                           count_launch();
      DSG_CUDA_CHECK(cudaMemcpyAsync(ground_truth, d, sizeof(double) * 3 * npix,
                                     cudaMemcpyDeviceToHost, ctx->stream));
      DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    }
    if (mask) {
      std::vector<uint8_t> m8(npix);
      DSG_CUDA_CHECK(cudaMemcpyAsync(m8.data(), views->mask.get() + npix * i, npix,
                                     cudaMemcpyDeviceToHost, ctx->stream));
      DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
      for (int64_t k = 0; k < npix; ++k) mask[k] = m8[k] ? 1.0 : 0.0;
    }
  });
}

int dsg_views_download_planar(dsg_ctx ctx, dsg_views views, int32_t i, float* gt_planar,
                              uint8_t* mask) {
  return guarded([&] {
    if (views->host) fail(kInvalidArgument, "host views are already in host memory");
    if (i < 0 || i >= views->n) fail(kInvalidArgument, "view index out of range");
    DeviceGuard g(ctx->device);
    const int64_t npix = (int64_t)views->width * views->height;
    if (gt_planar)
      DSG_CUDA_CHECK(cudaMemcpyAsync(gt_planar, views->gt.get() + 3 * npix * i,
                                     sizeof(float) * 3 * npix, cudaMemcpyDeviceToHost, ctx->stream));
    if (mask)
      DSG_CUDA_CHECK(cudaMemcpyAsync(mask, views->mask.get() + npix * i, npix,
                                     cudaMemcpyDeviceToHost, ctx->stream));
    DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  });
}

int dsg_view_order(uint64_t seed, int32_t n_views, int64_t iterations, int32_t* out) {
  return guarded([&] {  // trainer.hpp:157-163, 174
    if (n_views <= 0) fail(kNoViews, "training requires at least one view");
    std::vector<int32_t> order(n_views);
    std::iota(order.begin(), order.end(), 0);
    Rng vr(seed ^ 0x87aa11d3ULL);
    for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[(size_t)vr.below(i)]);
    for (int64_t it = 0; it < iterations; ++it) out[it] = order[(size_t)(it % n_views)];
  });
}

int dsg_views_create_host(dsg_ctx ctx, const dsg_camera* cams, const float* const* gt_planar,
                          const uint8_t* const* masks, int32_t n_views, dsg_views* out) {
  return guarded([&] {
    auto* v = new dsg_views_s();
    try {
      v->n = n_views;
      v->host = true;
      for (int32_t i = 0; i < n_views; ++i) {
        make_cam(&cams[i]);
        if (i == 0) {
          v->width = cams[0].width;
          v->height = cams[0].height;
        } else if (cams[i].width != v->width || cams[i].height != v->height) {
          fail(kDimensionMismatch, "all views must share one resolution");
        }
        v->cams.push_back(cams[i]);
        v->host_gt.push_back(gt_planar ? gt_planar[i] : nullptr);
        v->host_mask.push_back(masks ? masks[i] : nullptr);
      }
    } catch (...) {
      delete v;
      throw;
    }
    *out = v;
  });
}

int dsg_views_create_host_ref(dsg_ctx ctx, const dsg_camera* cams,
                              const double* const* ground_truth, const double* const* masks,
                              int32_t n_views, dsg_views* out) {
  return guarded([&] {
    auto* v = new dsg_views_s();
    try {
      v->n = n_views;
      v->host = true;
      v->ref_layout = true;
      for (int32_t i = 0; i < n_views; ++i) {
        make_cam(&cams[i]);
        if (i == 0) {
          v->width = cams[0].width;
          v->height = cams[0].height;
        } else if (cams[i].width != v->width || cams[i].height != v->height) {
          fail(kDimensionMismatch, "all views must share one resolution");
        }
        v->cams.push_back(cams[i]);
        v->host_gt.push_back(nullptr);
        v->host_mask.push_back(nullptr);
        v->host_gt64.push_back(ground_truth ? ground_truth[i] : nullptr);
        v->host_mask64.push_back(masks ? masks[i] : nullptr);
      }
    } catch (...) {
      delete v;
      throw;
    }
    *out = v;
  });
}

}  // extern "C"
namespace {
// One view from the reference's TrainView layout (HWC double ground truth, HW
// double mask) into the device's planar fp32 + byte-mask layout, on the host
// worker pool (read 32 B, write 13 B per pixel). mask >= 0.5 as k_mask_u8.
void convert_view_ref(const double* gt, const double* mask, int64_t npix, float* planar,
                      uint8_t* m8) {
  HostPool& pool = HostPool::get();
  const int64_t kMin = int64_t(1) << 15;
  const int64_t nt = std::min<int64_t>(pool.size() * 2, (npix + kMin - 1) / kMin);
  const int64_t per = (((npix + std::max<int64_t>(nt, 1) - 1) / std::max<int64_t>(nt, 1)) + 15) & ~int64_t(15);
  pool.run((int)((npix + per - 1) / per), [=](int k) {
    const int64_t p0 = (int64_t)k * per, p1 = std::min(npix, p0 + per);
    for (int64_t p = p0; p < p1; ++p) {
      planar[p] = (float)gt[3 * p];
      planar[npix + p] = (float)gt[3 * p + 1];
      planar[2 * npix + p] = (float)gt[3 * p + 2];
      m8[p] = mask[p] >= 0.5 ? 1 : 0;
    }
  });
}
}  // namespace
extern "C" {

int dsg_train(dsg_ctx ctx, dsg_model model, dsg_views views, const dsg_train_config* cfg,
              int32_t shards, dsg_progress_fn progress, void* user, double* final_loss,
              double* loss_trace) {
  return dsg_train_checkpointed(ctx, model, views, cfg, shards, progress, user, nullptr, nullptr,
                                final_loss, loss_trace);
}

int dsg_train_checkpointed(dsg_ctx ctx, dsg_model model, dsg_views views,
                           const dsg_train_config* cfg, int32_t shards, dsg_progress_fn progress,
                           void* user, dsg_checkpoint_fn checkpoint, void* ckpt_user,
                           double* final_loss, double* loss_trace) {
  return guarded([&] {
    validate_train(cfg);
    if (!views || views->n <= 0) fail(kNoViews, "training requires at least one view");
    if (shards < 1) fail(kInvalidArgument, "shards must be >= 1");
    if (final_loss) *final_loss = 0.0;
    ModelDev& m = model->m;
    if (cfg->iterations == 0) return;
    const int64_t iters = cfg->iterations;
    const int64_t until = (int64_t)(cfg->densify_stop_fraction * (double)iters);
    // DSG_FUSE_ADAM=0: separate chain and Adam launches (A/B; same bits)
    static const bool fuse_adam = [] {
      const char* e = std::getenv("DSG_FUSE_ADAM");
      return !(e && e[0] == '0');
    }();
    // Rng densify_rng(seed ^ 0xd3a51f11) (trainer.hpp:165): splitmix64 state
    // after the constructor's two warm-up draws (rng.hpp:25-30)
    uint64_t drng = (cfg->seed ^ 0xd3a51f11ULL) ^ 0x853c49e6748fea9bULL;
    drng += 2 * 0x9e3779b97f4a7c15ULL;
    RenderDev rd = make_rd(&cfg->render);
    std::vector<CamDev> cams;
    for (const auto& c : views->cams) cams.push_back(make_cam(&c));
    // seeded view order (trainer.hpp:157-163)
    std::vector<size_t> order(views->n);
    std::iota(order.begin(), order.end(), size_t{0});
    Rng vr(cfg->seed ^ 0x87aa11d3ULL);
    for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[(size_t)vr.below(i)]);
    if (views->host)
      for (int64_t it = 0; it < std::min<int64_t>(iters, views->n); ++it) {
        size_t vi = order[(size_t)it];
        const bool have = views->ref_layout ? views->host_gt64[vi] && views->host_mask64[vi]
                                            : views->host_gt[vi] && views->host_mask[vi];
        if (!have) fail(kInvalidArgument, "host view used by the schedule has no data");
      }

    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    reset_optimizer(ctx, m);   // fresh AdamState and stats (trainer.hpp:167-168)
    const int64_t npix = (int64_t)views->width * views->height;
    double* trace = ctx->loss_trace.ensure(iters);
    StageTimer& tm = ctx->timer;
    tm.on = ctx->profile;
    if (!ctx->timer_init) {
      for (int k = 0; k <= StageTimer::kStages; ++k) DSG_CUDA_CHECK(cudaEventCreate(&tm.ev[k]));
      DSG_CUDA_CHECK(cudaEventCreate(&ctx->ev_begin));
      DSG_CUDA_CHECK(cudaEventCreate(&ctx->ev_end));
      ctx->timer_init = true;
    }
    double stage[StageTimer::kStages] = {};
    if (views->host && !ctx->copy_stream) {
      DSG_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
      for (int k = 0; k < 2; ++k) {
        DSG_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->ev_copied[k], cudaEventDisableTiming));
        DSG_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->ev_consumed[k], cudaEventDisableTiming));
      }
    }
    // end-to-end mode: views come from pinned host memory, double-buffered
    // so the copy of step it+1 overlaps step it (slot reuse waits for the
    // loss of step it-1, the last reader of that slot)
    if (views->ref_layout && ctx->vpin_bytes < (size_t)(13 * npix)) {
      for (int k = 0; k < 2; ++k) {
        if (ctx->vpin[k]) DSG_CUDA_CHECK(cudaFreeHost(ctx->vpin[k]));
        DSG_CUDA_CHECK(cudaMallocHost(&ctx->vpin[k], (size_t)(13 * npix)));
      }
      ctx->vpin_bytes = (size_t)(13 * npix);
    }
    float* slot_gt = views->host ? ctx->vslot_gt.ensure(2 * 3 * (size_t)npix) : nullptr;
    uint8_t* slot_mask = views->host ? ctx->vslot_mask.ensure(2 * (size_t)npix) : nullptr;
    auto copy_view = [&](int64_t step) {
      const size_t v = order[(size_t)step % order.size()];
      const int slot = (int)(step & 1);
      cudaStream_t cs = ctx->copy_stream;
      const float* src_gt = views->host_gt[v];
      const uint8_t* src_mask = views->host_mask[v];
      if (views->ref_layout) {
        // reference-layout view: the slot's previous upload (step - 2) must
        // have left the pinned buffer before the host refills it; the GPU is
        // meanwhile still busy with the earlier steps' kernels
        DSG_CUDA_CHECK(cudaEventSynchronize(ctx->ev_copied[slot]));
        float* pf = reinterpret_cast<float*>(ctx->vpin[slot]);
        uint8_t* pm = reinterpret_cast<uint8_t*>(ctx->vpin[slot] + 12 * npix);
        convert_view_ref(views->host_gt64[v], views->host_mask64[v], npix, pf, pm);
        src_gt = pf;
        src_mask = pm;
      }
      DSG_CUDA_CHECK(cudaStreamWaitEvent(cs, ctx->ev_consumed[slot], 0));
      DSG_CUDA_CHECK(cudaMemcpyAsync(slot_gt + 3 * npix * slot, src_gt,
                                     sizeof(float) * 3 * npix, cudaMemcpyHostToDevice, cs));
      DSG_CUDA_CHECK(cudaMemcpyAsync(slot_mask + npix * slot, src_mask, npix,
                                     cudaMemcpyHostToDevice, cs));
      DSG_CUDA_CHECK(cudaEventRecord(ctx->ev_copied[slot], cs));
    };
    DSG_CUDA_CHECK(cudaEventRecord(ctx->ev_begin, st));
    if (views->host) {
      // slots are free once the previous call's stream work is done
      for (int k = 0; k < 2; ++k) DSG_CUDA_CHECK(cudaEventRecord(ctx->ev_consumed[k], st));
      copy_view(0);
    }
    for (int64_t it = 0; it < iters; ++it) {
      const size_t vi = order[(size_t)it % order.size()];
      const CamDev& cam = cams[vi];
      const int slot = (int)(it & 1);
      const float* gt = views->host ? slot_gt + 3 * npix * (size_t)slot
                                    : views->gt.get() + 3 * npix * vi;
      const uint8_t* mk = views->host ? slot_mask + npix * (size_t)slot
                                      : views->mask.get() + npix * vi;
      if (views->host) {
        DSG_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_copied[slot], 0));
        if (it + 1 < iters) copy_view(it + 1);
      }
      bin_frame(ctx->frame, m.params.get(), m.cap, m.n, cam, rd, st, &tm);
      Frame& f = ctx->frame;
      const bool empty = f.n_visible == 0 || f.n_dup == 0;
      if (empty) {
        for (int k = 1; k <= 4; ++k) tm.mark(k, st);
        forward(ctx, m, cam, rd);
      } else {
        blend_forward(f, m.params.get(), m.cap, cam, rd, st);
      }
      tm.mark(5, st);
      masked_loss_dev(f, gt, mk, views->width, views->height, cfg->loss_lambda, st, trace + it);
      if (views->host)  // view slot free for the upload two steps ahead
        DSG_CUDA_CHECK(cudaEventRecord(ctx->ev_consumed[slot], st));
      tm.mark(6, st);
      const double decay = std::pow(cfg->lr_mu_decay, (double)it / (double)iters);
      const double rates[5] = {cfg->lr_mu * decay, cfg->lr_scale, cfg->lr_rot, cfg->lr_opacity,
                               cfg->lr_color};
      if (!empty) blend_backward(f, m.params.get(), m.cap, cam, rd, st);
      tm.mark(7, st);
      if (empty) {
        DSG_CUDA_CHECK(cudaMemsetAsync(m.grads.get(), 0, sizeof(float) * kParams * m.cap, st));
        DSG_CUDA_CHECK(cudaMemsetAsync(m.touch.get(), 0, sizeof(int32_t) * m.cap, st));
        DSG_CUDA_CHECK(cudaMemsetAsync(m.dmean.get(), 0, sizeof(float) * 2 * m.cap, st));
      } else {
        ChainArgs a;
        a.params = m.params.get();
        a.pitch = m.cap;
        a.n = m.n;
        a.cam = cam;
        a.tcount = f.tcount.get();
        a.dup_base = f.dup_base.get();
        a.partials = f.partials.get();
        a.n_dup = f.n_dup;
        a.tmask = f.tmask.get();
        a.grads = m.grads.get();
        a.dmean = m.dmean.get();
        a.touch = m.touch.get();
        if (fuse_adam) {
          m.adam_step += 1;  // chain + Adam in one pass (no gradient store)
          chain_adam(a, make_adam(m, rates, cfg->adam, m.adam_step, true), st);
        } else {
          chain_3d(a, st);
        }
      }
      tm.mark(8, st);
      if (empty || !fuse_adam) {
        m.adam_step += 1;
        adam_update(make_adam(m, rates, cfg->adam, m.adam_step, true), st);
      }
      m.iteration += 1;
      // densify at (it+1) % interval == 0 while (it+1) < stop (trainer.hpp:195-202)
      if (cfg->densify_interval > 0 && (it + 1) % cfg->densify_interval == 0 && (it + 1) < until)
        densify_dev(m, ctx->spare, ctx->dscratch, cfg->prune_opacity, cfg->densify_grad_threshold,
                    cfg->split_scale_threshold, drng, ctx->frame.scan, st);
      tm.mark(9, st);
      if (tm.on) {
        DSG_CUDA_CHECK(cudaEventSynchronize(tm.ev[9]));
        float ms;
        for (int s = 0; s < StageTimer::kStages; ++s) {
          DSG_CUDA_CHECK(cudaEventElapsedTime(&ms, tm.ev[s], tm.ev[s + 1]));
          stage[s] += ms;
        }
      }
      // CheckpointSink at the interval, then ProgressSink (trainer.hpp:204-207);
      // the callback may read the model and its Adam moments through the ABI
      const bool ckpt_now = checkpoint && cfg->checkpoint_interval > 0 &&
                            (it + 1) % cfg->checkpoint_interval == 0;
      if (progress || ckpt_now) {
        double l;
        DSG_CUDA_CHECK(cudaMemcpyAsync(&l, trace + it, sizeof(double), cudaMemcpyDeviceToHost, st));
        DSG_CUDA_CHECK(cudaStreamSynchronize(st));
        if (ckpt_now) checkpoint(m.iteration, l, model, ckpt_user);
        if (progress) progress(it + 1, l, user);
      }
    }
    DSG_CUDA_CHECK(cudaEventRecord(ctx->ev_end, st));
    DSG_CUDA_CHECK(cudaEventSynchronize(ctx->ev_end));
    float total;
    DSG_CUDA_CHECK(cudaEventElapsedTime(&total, ctx->ev_begin, ctx->ev_end));
    ctx->last_total_ms = total;
    ctx->last_iters = iters;
    for (int s = 0; s < StageTimer::kStages; ++s) ctx->last_stage_ms[s] = stage[s];
    std::vector<double> tr(iters);
    DSG_CUDA_CHECK(cudaMemcpy(tr.data(), trace, sizeof(double) * iters, cudaMemcpyDeviceToHost));
    if (final_loss) *final_loss = tr.back();
    if (loss_trace) std::memcpy(loss_trace, tr.data(), sizeof(double) * iters);
    if (checkpoint) checkpoint(m.iteration, tr.back(), model, ckpt_user);  // trainer.hpp:209
  });
}

int dsg_set_exact_masks(int32_t enable) {
  g_exact_masks.store(enable != 0);
  return 0;
}

int dsg_set_profiling(dsg_ctx ctx, int32_t enable) {
  return guarded([&] { ctx->profile = enable != 0; });
}

int dsg_render_mask(dsg_ctx ctx, const double* points, int64_t n, const dsg_camera* cam_in,
                    double footprint_px, double dilation_px, double* mask) {
  return guarded([&] {
    // render.hpp:212-214: footprint check, then camera validation
    if (footprint_px < 0.5) fail(kInvalidArgument, "footprint_px must be >= 0.5");
    CamDev cam = make_cam(cam_in);
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    const int64_t npix = (int64_t)cam.width * cam.height;
    uint8_t* m8 = ctx->stage_u8.ensure(npix);
    DSG_CUDA_CHECK(cudaMemsetAsync(m8, 0, npix, st));
    if (n > 0) {
      double* d = ctx->stage_d2.ensure(3 * n);
      DSG_CUDA_CHECK(cudaMemcpyAsync(d, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
      render_mask_dev(d, n, cam, footprint_px + dilation_px, m8, st);
    }
    std::vector<uint8_t> h(npix);
    DSG_CUDA_CHECK(cudaMemcpyAsync(h.data(), m8, npix, cudaMemcpyDeviceToHost, st));
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < npix; ++i) mask[i] = h[i] ? 1.0 : 0.0;
  });
}

int dsg_views_synthesize(dsg_ctx ctx, dsg_model gt_model, const dsg_render_config* cfg,
                         const dsg_camera* cams, int32_t n_views, const double* points,
                         int64_t n_points, int32_t use_masks, double footprint_px,
                         double dilation_px, dsg_views* out) {
  return guarded([&] {
    RenderDev rd = make_rd(cfg);
    if (use_masks && footprint_px < 0.5) fail(kInvalidArgument, "footprint_px must be >= 0.5");
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    auto* v = new dsg_views_s();
    try {
      v->n = n_views;
      if (n_views > 0) {
        v->width = cams[0].width;
        v->height = cams[0].height;
      }
      const int64_t npix = (int64_t)v->width * v->height;
      v->gt.ensure(std::max<int64_t>(1, 3 * npix * n_views));
      v->mask.ensure(std::max<int64_t>(1, npix * n_views));
      double* dpts = nullptr;
      if (use_masks && n_points > 0) {
        dpts = ctx->stage_d2.ensure(3 * n_points);
        DSG_CUDA_CHECK(cudaMemcpyAsync(dpts, points, sizeof(double) * 3 * n_points,
                                       cudaMemcpyHostToDevice, st));
      }
      for (int32_t i = 0; i < n_views; ++i) {
        CamDev cam = make_cam(&cams[i]);
        if (cams[i].width != v->width || cams[i].height != v->height)
          fail(kDimensionMismatch, "all views must share one resolution");
        v->cams.push_back(cams[i]);
        forward(ctx, gt_model->m, cam, rd);  // ground truth = render(gt_model) (runtime.hpp:195)
        DSG_CUDA_CHECK(cudaMemcpyAsync(v->gt.get() + 3 * npix * i, ctx->frame.rgb.get(),
                                       sizeof(float) * 3 * npix, cudaMemcpyDeviceToDevice, st));
        uint8_t* mi = v->mask.get() + npix * i;
        if (use_masks) {
          DSG_CUDA_CHECK(cudaMemsetAsync(mi, 0, npix, st));
          if (n_points > 0) render_mask_dev(dpts, n_points, cam, footprint_px + dilation_px, mi, st);
        } else {
          DSG_CUDA_CHECK(cudaMemsetAsync(mi, 1, npix, st));
        }
      }
      DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    } catch (...) {
      delete v;
      throw;
    }
    *out = v;
  });
}

int dsg_knn_mean(dsg_ctx ctx, const double* points, int64_t n, int32_t k, double* out) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    if (n <= 0) return;
    double* d = ctx->stage_d2.ensure(4 * n);
    DSG_CUDA_CHECK(cudaMemcpyAsync(d, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, ctx->stream));
    knn_mean_dev(points, d, n, k, d + 3 * n, ctx->frame.sort, ctx->stream);
    DSG_CUDA_CHECK(cudaMemcpyAsync(out, d + 3 * n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  });
}

int dsg_median_nn_spacing(dsg_ctx ctx, const double* points, int64_t n, double* out) {
  return guarded([&] {  // seed.hpp:39-45
    if (n <= 0) fail(kEmptyCloud, "empty point cloud");
    if (n == 1) {
      *out = 1.0;
      return;
    }
    std::vector<double> nn(n);
    DeviceGuard g(ctx->device);
    double* d = ctx->stage_d2.ensure(4 * n);
    DSG_CUDA_CHECK(cudaMemcpyAsync(d, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, ctx->stream));
    knn_mean_dev(points, d, n, 1, d + 3 * n, ctx->frame.sort, ctx->stream);
    DSG_CUDA_CHECK(cudaMemcpyAsync(nn.data(), d + 3 * n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    std::nth_element(nn.begin(), nn.begin() + n / 2, nn.end());
    *out = nn[(size_t)(n / 2)];
  });
}

int dsg_seed_gaussians(dsg_ctx ctx, const double* points, const double* colors, int64_t n,
                       int32_t rule, int32_t k, double fixed_scale, dsg_model model) {
  return guarded([&] {  // seed.hpp:49-74
    if (n <= 0) fail(kEmptyCloud, "cannot seed from an empty cloud");
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    ModelDev& m = model->m;
    m.reserve(n);
    m.n = n;
    m.iteration = 0;
    m.origin_partition = -1;
    double* d = ctx->stage_d2.ensure(7 * n);
    DSG_CUDA_CHECK(cudaMemcpyAsync(d, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
    DSG_CUDA_CHECK(cudaMemcpyAsync(d + 3 * n, colors, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
    const double* scale = nullptr;
    if (rule == 0 && n > 1) {
      knn_mean_dev(points, d, n, k, d + 6 * n, ctx->frame.sort, st);
      scale = d + 6 * n;
    }
    const double op = std::log(0.1 / (1.0 - 0.1));
    seed_params_dev(d, d + 3 * n, scale, n, std::log(fixed_scale), op, m.params.get(), m.cap, st);
    reset_optimizer(ctx, m);
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

int dsg_ground_truth_model(dsg_ctx ctx, const double* points, const double* colors, int64_t n,
                           double scale, double opacity, dsg_model model) {
  return guarded([&] {  // seed.hpp:78-94
    if (n <= 0) fail(kEmptyCloud, "cannot build ground truth from nothing");
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    ModelDev& m = model->m;
    m.reserve(n);
    m.n = n;
    m.iteration = 0;
    m.origin_partition = -1;
    double* d = ctx->stage_d2.ensure(6 * n);
    DSG_CUDA_CHECK(cudaMemcpyAsync(d, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
    DSG_CUDA_CHECK(cudaMemcpyAsync(d + 3 * n, colors, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
    seed_params_dev(d, d + 3 * n, nullptr, n, std::log(std::max(scale, 1e-7)),
                    std::log(opacity / (1.0 - opacity)), m.params.get(), m.cap, st);
    reset_optimizer(ctx, m);
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

int64_t dsg_launch_count(void) { return g_launches.load(); }

int dsg_nvtx_push(const char* name) {
  nvtxRangePushA(name ? name : "dsg");
  return 0;
}
int dsg_nvtx_pop(void) {
  nvtxRangePop();
  return 0;
}

int dsg_frame_work(dsg_ctx ctx, int64_t* composited, int64_t* term_fixups,
                   int64_t* term_changed) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    int64_t c = 0, f = 0, ch = 0;
    frame_work_dev(ctx->frame, ctx->stream, &c, &f, &ch);
    if (composited) *composited = c;
    if (term_fixups) *term_fixups = f;
    if (term_changed) *term_changed = ch;
  });
}

int dsg_frame_stats(dsg_ctx ctx, int64_t* n_visible, int64_t* n_dup) {
  return guarded([&] {
    if (n_visible) *n_visible = ctx->frame.n_visible;
    if (n_dup) *n_dup = ctx->frame.n_dup;
  });
}

int dsg_render_timed(dsg_ctx ctx, dsg_model model, const dsg_camera* cams, int32_t n,
                     const dsg_render_config* cfg, int32_t repeats, double* ms) {
  return guarded([&] {
    RenderDev rd = make_rd(cfg);
    std::vector<CamDev> cv;
    for (int32_t i = 0; i < n; ++i) cv.push_back(make_cam(&cams[i]));
    DeviceGuard g(ctx->device);
    cudaEvent_t a, b;
    DSG_CUDA_CHECK(cudaEventCreate(&a));
    DSG_CUDA_CHECK(cudaEventCreate(&b));
    DSG_CUDA_CHECK(cudaEventRecord(a, ctx->stream));
    for (int32_t r = 0; r < repeats; ++r)
      for (const CamDev& c : cv) forward(ctx, model->m, c, rd);
    DSG_CUDA_CHECK(cudaEventRecord(b, ctx->stream));
    DSG_CUDA_CHECK(cudaEventSynchronize(b));
    float t;
    DSG_CUDA_CHECK(cudaEventElapsedTime(&t, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *ms = t;
  });
}

int dsg_heightfield_cloud(dsg_ctx ctx, int64_t n, uint64_t seed, double span, double amp,
                          double spikes, int32_t nmodes, const double* modes, double* positions,
                          double* colors, double* normals) {
  return guarded([&] {
    if (n <= 0) fail(kEmptyCloud, "empty cloud");
    if (nmodes < 0 || (nmodes > 0 && !modes)) fail(kInvalidArgument, "bad mode table");
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    // generated in slices so the device scratch stays bounded at any size
    const int64_t slice = int64_t(1) << 24;
    DevBuf<double> buf;
    buf.ensure(9 * (size_t)std::min(n, slice));
    for (int64_t s0 = 0; s0 < n; s0 += slice) {
      const int64_t m = std::min(slice, n - s0);
      heightfield_slice_dev(n, s0, m, seed, span, amp, spikes, nmodes, modes, buf.get(),
                            buf.get() + 3 * m, buf.get() + 6 * m, st);
      if (positions)
        DSG_CUDA_CHECK(cudaMemcpyAsync(positions + 3 * s0, buf.get(), sizeof(double) * 3 * m,
                                       cudaMemcpyDeviceToHost, st));
      if (colors)
        DSG_CUDA_CHECK(cudaMemcpyAsync(colors + 3 * s0, buf.get() + 3 * m, sizeof(double) * 3 * m,
                                       cudaMemcpyDeviceToHost, st));
      if (normals)
        DSG_CUDA_CHECK(cudaMemcpyAsync(normals + 3 * s0, buf.get() + 6 * m, sizeof(double) * 3 * m,
                                       cudaMemcpyDeviceToHost, st));
      DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    }
  });
}

int dsg_image_metrics(dsg_ctx ctx, const double* a, const double* b, int32_t width,
                      int32_t height, double* psnr, double* ssim) {
  return guarded([&] {  // psnr / ssim (metrics.hpp:20-38) of two HWC double RGB images
    if (!a || !b || width <= 0 || height <= 0) fail(kDimensionMismatch, "image shapes differ");
    if (ssim && (width < 11 || height < 11))
      fail(kTooSmall, "images must be at least 11 px per side");
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    const int64_t npix = (int64_t)width * height;
    double* d = ctx->stage_d.ensure(6 * npix);
    float* f = ctx->stage_f.ensure(6 * npix);
    DSG_CUDA_CHECK(cudaMemcpyAsync(d, a, sizeof(double) * 3 * npix, cudaMemcpyHostToDevice, st));
    DSG_CUDA_CHECK(cudaMemcpyAsync(d + 3 * npix, b, sizeof(double) * 3 * npix,
                                   cudaMemcpyHostToDevice, st));
    k_aos_to_planar<<<nblk(npix), 256, 0, st>>>(d, npix, 3, f, npix);
    k_aos_to_planar<<<nblk(npix), 256, 0, st>>>(d + 3 * npix, npix, 3, f + 3 * npix, npix);
    count_launch(2);
    double* out = ctx->frame.loss_out.ensure(2);
    image_metrics_dev(ctx->frame, f, f + 3 * npix, width, height, st, out);
    double h[2];
    DSG_CUDA_CHECK(cudaMemcpyAsync(h, out, sizeof h, cudaMemcpyDeviceToHost, st));
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    if (psnr) *psnr = h[0];
    if (ssim) *ssim = h[1];
  });
}

int dsg_eval_view(dsg_ctx ctx, dsg_model model, dsg_model truth, const dsg_camera* cam_in,
                  const dsg_render_config* cfg, double* psnr, double* ssim) {
  return guarded([&] {  // runtime.hpp:483-492: psnr/ssim of render(merged) vs render(gt)
    RenderDev rd = make_rd(cfg);
    CamDev cam = make_cam(cam_in);
    if (cam.width < 11 || cam.height < 11) fail(kTooSmall, "images must be at least 11 px per side");
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    const int64_t npix = (int64_t)cam.width * cam.height;
    forward(ctx, truth->m, cam, rd);
    float* t = ctx->stage_f.ensure(3 * npix);
    DSG_CUDA_CHECK(cudaMemcpyAsync(t, ctx->frame.rgb.get(), sizeof(float) * 3 * npix,
                                   cudaMemcpyDeviceToDevice, st));
    forward(ctx, model->m, cam, rd);
    double* out = ctx->frame.loss_out.ensure(2);
    image_metrics_dev(ctx->frame, ctx->frame.rgb.get(), t, cam.width, cam.height, st, out);
    double h[2];
    DSG_CUDA_CHECK(cudaMemcpyAsync(h, out, sizeof h, cudaMemcpyDeviceToHost, st));
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    if (psnr) *psnr = h[0];
    if (ssim) *ssim = h[1];
  });
}

int dsg_host_register(void* ptr, int64_t bytes) {
  return guarded([&] { DSG_CUDA_CHECK(cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault)); });
}

int dsg_host_unregister(void* ptr) {
  return guarded([&] { DSG_CUDA_CHECK(cudaHostUnregister(ptr)); });
}

int dsg_partition(dsg_ctx ctx, const double* positions, int64_t n, int32_t nparts, double margin,
                  int32_t* axis, double* cut_lo, double* cut_hi, double* owned_box,
                  int64_t* owned_count, int64_t* ghost_count, uint32_t* owned_idx,
                  uint32_t* ghost_idx, int64_t cap) {
  return guarded([&] {  // partition.hpp:42-104
    DeviceGuard g(ctx->device);
    PartitionResult r = partition_dev(positions, n, nparts, margin, ctx->frame.sort,
                                      ctx->frame.scan, ctx->stream);
    *axis = r.axis;
    int64_t oi = 0, gi = 0;
    for (int k = 0; k < nparts; ++k) {
      cut_lo[k] = r.cut_lo[k];
      cut_hi[k] = r.cut_hi[k];
      for (int c = 0; c < 6; ++c) owned_box[6 * k + c] = r.box[6 * k + c];
      owned_count[k] = (int64_t)r.owned[k].size();
      ghost_count[k] = (int64_t)r.ghost[k].size();
      if (!owned_idx || !ghost_idx) continue;  // size query
      for (uint32_t x : r.owned[k]) {
        if (oi < cap) owned_idx[oi] = x;
        ++oi;
      }
      for (uint32_t x : r.ghost[k]) {
        if (gi < cap) ghost_idx[gi] = x;
        ++gi;
      }
    }
    if (owned_idx && ghost_idx && (oi > cap || gi > cap))
      fail(kInvalidArgument, "index capacity too small");
  });
}

int dsg_merge_models(dsg_ctx ctx, const dsg_model* models, int32_t nparts, int32_t axis,
                     const double* cut_lo, const double* cut_hi, dsg_model out) {
  return guarded([&] {  // merge_models (partition.hpp:109-126), single process
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    std::vector<MergeSrc> src(nparts);
    int64_t it = 0;
    for (int k = 0; k < nparts; ++k) {
      const ModelDev& m = models[k]->m;
      src[k] = {m.params.get(), m.cap, m.n, cut_lo[k], cut_hi[k]};
      it = std::max(it, m.iteration);
    }
    std::vector<int64_t> cnt(nparts);
    merge_trim_count(src.data(), nparts, axis, ctx->merge, ctx->frame.scan, st, cnt.data());
    int64_t total = 0;
    for (int k = 0; k < nparts; ++k) total += cnt[k];
    ModelDev& o = out->m;
    o.reserve(std::max<int64_t>(total, 1));
    o.n = total;
    o.iteration = it;
    o.origin_partition = -1;
    int64_t off = 0;
    for (int k = 0; k < nparts; ++k) {
      merge_trim_scatter(src[k], k, ctx->merge, o.params.get(), o.cap, off, st);
      off += cnt[k];
    }
    reset_optimizer(ctx, o);
    DSG_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

struct dsg_comm_s {
  void* nccl = nullptr;      // 64 CTAs per collective: the merge exchange
  void* nccl_p2p = nullptr;  // NCCL's default CTAs: the band gather
  int nranks = 1, rank = 0;
  std::vector<int> band_rows;  // first tile row of each rank's band, last distributed render
};

int dsg_comm_unique_id(uint8_t* out128) {
  return guarded([&] { nccl_unique_id(out128); });
}

int dsg_comm_create(dsg_ctx ctx, const uint8_t* id128, int32_t nranks, int32_t rank,
                    dsg_comm* out) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    auto* c = new dsg_comm_s();
    c->nranks = nranks;
    c->rank = rank;
    c->nccl = nccl_comm_init(id128, nranks, rank);
    c->nccl_p2p = nccl_comm_split_default(c->nccl, rank);
    *out = c;
  });
}

int dsg_comm_destroy(dsg_comm comm) {
  return guarded([&] {
    if (!comm) return;
    if (comm->nccl_p2p) nccl_comm_destroy(comm->nccl_p2p);
    nccl_comm_destroy(comm->nccl);
    delete comm;
  });
}

int dsg_merge_allgather_multi(dsg_ctx ctx, dsg_comm comm, const dsg_model* locals,
                              int32_t nlocal, int32_t axis, const double* cut_lo,
                              const double* cut_hi, dsg_model merged, int64_t* n_merged,
                              double* ms) {
  return guarded([&] {
    if (nlocal < 1 || !locals) fail(kInvalidArgument, "no local partitions");
    DeviceGuard g(ctx->device);
    std::vector<const ModelDev*> ms_(nlocal);
    for (int j = 0; j < nlocal; ++j) ms_[j] = &locals[j]->m;
    float t = 0.f;  // device time of the survivor exchange (the NCCL all-gathers)
    int64_t it_max = 0;
    const int64_t total = merge_allgather_dev(comm->nccl, comm->nranks, comm->rank, ms_.data(),
                                              nlocal, axis, cut_lo, cut_hi, merged->m,
                                              ctx->frame.scan, ctx->merge, ctx->stream, &t,
                                              &it_max);
    merged->m.iteration = it_max;  // merge_models: iteration = max (partition.hpp:124)
    merged->m.origin_partition = -1;
    reset_optimizer(ctx, merged->m);
    DSG_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    if (n_merged) *n_merged = total;
    if (ms) *ms = t;
  });
}

const char* dsg_merge_exchange(void) { return dsg::g_merge_path; }

int dsg_comm_bench_allgather(dsg_ctx ctx, dsg_comm comm, int64_t bytes, int32_t reps,
                             double* ms) {
  return guarded([&] {
    if (!comm || bytes < 4 || reps < 1) fail(kInvalidArgument, "bench_allgather: bad arguments");
    DeviceGuard g(ctx->device);
    const double t = bench_allgather_dev(comm->nccl, comm->nranks, bytes, reps, ctx->stream);
    if (ms) *ms = t;
  });
}

int dsg_merge_allgather(dsg_ctx ctx, dsg_comm comm, dsg_model local, int32_t axis, double cut_lo,
                        double cut_hi, dsg_model merged, int64_t* n_merged, double* ms) {
  return dsg_merge_allgather_multi(ctx, comm, &local, 1, axis, &cut_lo, &cut_hi, merged, n_merged,
                                   ms);
}

int dsg_render_distributed(dsg_ctx ctx, dsg_comm comm, dsg_model model, const dsg_camera* cam_in,
                           const dsg_render_config* cfg, double* rgb, double* ms) {
  return guarded([&] {
    RenderDev rd = make_rd(cfg);
    CamDev cam = make_cam(cam_in);
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    const int R = comm ? comm->nranks : 1, me = comm ? comm->rank : 0;
    cudaEvent_t a, b;
    DSG_CUDA_CHECK(cudaEventCreate(&a));
    DSG_CUDA_CHECK(cudaEventCreate(&b));
    DSG_CUDA_CHECK(cudaEventRecord(a, st));
    // Bands of tile rows balanced by splat count: every
    // rank histograms the replicated model's projected centres per tile row
    // (integer atomics: identical on every rank, no exchange) and cuts the
    // rows at the R-quantiles of that count.
    std::vector<int> t0(R), t1(R), r0(R), r1(R);
    t0[0] = 0;
    t1[R - 1] = cam.tiles_y;
    if (R > 1) {
      uint32_t* hist = ctx->frame.row_hist.ensure(cam.tiles_y);
      center_row_hist_dev(model->m.params.get(), model->m.cap, model->m.n, cam, hist, st);
      std::vector<uint32_t> h(cam.tiles_y);
      DSG_CUDA_CHECK(cudaMemcpyAsync(h.data(), hist, sizeof(uint32_t) * cam.tiles_y,
                                     cudaMemcpyDeviceToHost, st));
      DSG_CUDA_CHECK(cudaStreamSynchronize(st));
      int64_t total = 0;
      for (uint32_t v : h) total += v;
      int64_t run = 0;
      int row = 0;
      for (int r = 1; r < R; ++r) {  // first row whose prefix reaches r/R of the splats
        const int64_t want = total * r / R;
        while (row < cam.tiles_y && run + h[row] <= want) run += h[row++];
        // keep every band non-empty and increasing
        const int lo = t0[r - 1] + 1, hi = cam.tiles_y - (R - r);
        t0[r] = std::min(std::max(row, lo), hi);
        t1[r - 1] = t0[r];
      }
    }
    for (int r = 0; r < R; ++r) {
      r0[r] = std::min(t0[r] * kTile, cam.height);
      r1[r] = std::min(t1[r] * kTile, cam.height);
    }
    if (comm) comm->band_rows.assign(t0.begin(), t0.end());
    CamDev band = cam;
    band.band_ty0 = t0[me];
    band.band_ty1 = t1[me];
    forward(ctx, model->m, band, rd);
    if (R > 1) gather_bands_dev(comm->nccl_p2p ? comm->nccl_p2p : comm->nccl, R, me, ctx->frame.rgb.get(), cam.width, cam.height, r0, r1, st);
    DSG_CUDA_CHECK(cudaEventRecord(b, st));
    DSG_CUDA_CHECK(cudaEventSynchronize(b));
    float t;
    DSG_CUDA_CHECK(cudaEventElapsedTime(&t, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (ms) *ms = t;
    if (rgb && me == 0) {
      const int64_t npix = (int64_t)cam.width * cam.height;
      double* d = ctx->stage_d.ensure(4 * npix);
      k_render_out<<<nblk(npix), 256, 0, st>>>(ctx->frame.rgb.get(), ctx->frame.T.get(), npix, d,
                                                d + 3 * npix);
      count_launch();
      DSG_CUDA_CHECK(cudaMemcpyAsync(rgb, d, sizeof(double) * 3 * npix, cudaMemcpyDeviceToHost, st));
      DSG_CUDA_CHECK(cudaStreamSynchronize(st));
    }
  });
}

int dsg_last_timing(dsg_ctx ctx, double* total_ms, double* stage_ms) {
  return guarded([&] {
    if (total_ms) *total_ms = ctx->last_total_ms;
    if (stage_ms)
      for (int s = 0; s < StageTimer::kStages; ++s) stage_ms[s] = ctx->last_stage_ms[s];
  });
}

}  // extern "C"
