// Raster pipeline state for one view (per context scratch) and launchers.
#pragma once
#include <deque>
#include <atomic>

#include "dsg_internal.h"

namespace dsg {

// Blend work units split a tile list only when it is long enough to form
// the kernel's tail: segment length = max(kSegMin, n_dup / kSegDiv), i.e. a
// list longer than the average work of ~kSegDiv/8 concurrent warps.
#ifndef DSG_SEG_MIN
#define DSG_SEG_MIN 256
#endif
constexpr int kSegMin = DSG_SEG_MIN;
#ifndef DSG_SEG_DIV
#define DSG_SEG_DIV 8192
#endif
constexpr int kSegDiv = DSG_SEG_DIV;
constexpr int kUnitPlanes = 15;  // per-unit per-pixel planes (blend.cu UnitPlane)
#ifndef DSG_SPLIT_MIN
#define DSG_SPLIT_MIN 32768
#endif
#ifndef DSG_SPLIT_FACTOR
#define DSG_SPLIT_FACTOR 4
#endif
// the forward splits lists longer than max(kSplitMin, kSplitFactor * seg_len)
constexpr int64_t kSplitMin = DSG_SPLIT_MIN;
constexpr int64_t kSplitFactor = DSG_SPLIT_FACTOR;

struct PreprocessArgs {
  const float* params;  // [14][pitch] planar fp32 model
  int64_t pitch, n;
  CamDev cam;
  RenderDev rd;
  float4* rec;          // [n][3] blend payload (model order)
  int4* trect;          // [n] pixel rect (x0, y0, x1, y1), render.hpp:71-81
  int4* erect;          // [n] effective (alpha >= cutoff) rect, widened by 1 px
  float4* mrow;         // [n] sub-tile mask constants (ixy/ixx, 1/ixx, q0, qcut)
  uint32_t* tcount;     // [n] overlapped tiles (0 = culled)
  double* depth;        // [n] camera-space depth (fp64)
  double2* exact;       // [n][3] fp64 (mx,my) (ixx,ixy) (iyy,op) for the guard band
  unsigned long long* drange;  // [2] fp64 depth min / max bits of the visible set
};

// Scratch for one rendered view: binning products, per-pixel forward state,
// loss buffers and backward partials.
struct Frame {
  int64_t n = 0, n_visible = 0, n_dup = 0, tiles = 0;
  int width = 0, height = 0;
  // per gaussian (model order)
  DevBuf<float4> rec;
  DevBuf<int4> trect, erect;
  DevBuf<float4> mrow;        // sub-tile mask row-interval constants
  DevBuf<uint32_t> tcount, dup_base;
  DevBuf<double> depth;
  DevBuf<double2> exact;     // [n][3] fp64 mean2d, conic, opacity
  // visible set, depth-sorted
  DevBuf<uint32_t> vis_key, vis_idx, vis_key2, vis_idx2, offs;
  DevBuf<uint32_t> vslot;        // visible-slot scan (order-preserving compaction)
  DevBuf<unsigned long long> drange;
  DevBuf<uint32_t> long_runs, run_vals;  // long equal-key runs needing a radix sort
  DevBuf<unsigned long long> run_keys;
  uint32_t* sorted_idx = nullptr;
  // duplicates
  DevBuf<uint32_t> tile_key, dup_val, tile_key2, dup_val2;
  uint32_t* sorted_tile = nullptr;
  uint32_t* sorted_val = nullptr;
  DevBuf<uint2> ranges;
  DevBuf<uint8_t> emask;      // per sorted entry: touched 8x4 sub-tiles of its tile
  DevBuf<uint32_t> tile_order, tile_bins;  // longest-first blend schedule (band tiles)
  // blend work units: (tile, <= seg_len entries), tiles in longest-first order
  DevBuf<uint4> units;
  DevBuf<uint32_t> unit_base;  // [band tiles + 1] first unit of each ordered tile; [nt] = total
  DevBuf<uint32_t> nonlast;    // units that are not their tile's last segment
  DevBuf<float> ubuf;          // per unit, per pixel segment state (blend.cu UnitPlane)
  int64_t unit_cap = 0, band_tiles = 0, seg_len = kSegMin, split_len = 0, split_cap = 0;
  DevBuf<uint32_t> counters;
  DevBuf<uint32_t> amb, tile_unit;  // termination fix-up: flagged pixels, tile -> first unit
  DevBuf<unsigned long long> work;  // frame_work_dev scratch
  DevBuf<uint32_t> term_base, term_ntask;  // termination fix-up tasks (blend.cu)
  DevBuf<uint2> term_task;
  DevBuf<uint8_t> term_rec;
  DevBuf<uint32_t> row_hist;        // splats per tile row (render band balancing)
  // per pixel (planar fp32)
  DevBuf<float> rgb, T, dL, Tband;
  DevBuf<uint32_t> last;
  DevBuf<int32_t> ncontrib;
  // backward partials: [n_dup][8 sub-tiles][8] (values 0..7) then [n_dup][8] (value 8)
  DevBuf<float> partials;
  DevBuf<uint32_t> tmask;     // 8-bit touched-sub-tile mask per duplicate, 4 per word
  // device copy of the blend kernels' guard-band context (read by the rare
  // fp64 path through a pointer, so it never lands on the thread stack)
  DevBuf<uint8_t> evalctx;
  // loss scratch
  DevBuf<double> ssim_pqr, loss_parts;
  DevBuf<uint32_t> loss_counts;
  DevBuf<double> loss_out;
  DevBuf<uint8_t> ones_mask;  // all-ones mask (unmasked SSIM metric)
  SortScratch sort;
  ScanScratch scan;
  // high-priority side stream for the split-tile forward, which runs beside
  // the main forward kernel (created on first use, on the frame's device)
  struct Side {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    cudaStream_t get() {
      if (!s) {
        int lo = 0, hi = 0;
        DSG_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        DSG_CUDA_CHECK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi));
        DSG_CUDA_CHECK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        DSG_CUDA_CHECK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
      }
      return s;
    }
    Side() = default;
    Side(const Side&) = delete;
    Side& operator=(const Side&) = delete;
    ~Side() {
      if (s) {
        cudaEventDestroy(fork);
        cudaEventDestroy(join);
        cudaStreamDestroy(s);
      }
    }
  } side;
};

// Model tensors on device (planar [14][cap] fp32 for params/grads/moments).
struct ModelDev {
  int64_t n = 0, cap = 0;
  int64_t iteration = 0;
  int32_t origin_partition = -1;
  int64_t adam_step = 0;
  DevBuf<float> params, grads, m, v, dmean;
  DevBuf<double> stat_norm;  // screen_grad_norm (gradient.hpp:16), fp64 like the reference
  DevBuf<int32_t> touch, stat_count;
  void reserve(int64_t c);
};

struct ChainArgs {
  const float* params;
  int64_t pitch, n;
  CamDev cam;
  const uint32_t* tcount;
  const uint32_t* dup_base;
  const float* partials;    // blend.cu layout: [n_dup][8][8] then [n_dup][8]
  int64_t n_dup;
  const uint32_t* tmask;
  float* grads;     // [14][pitch]
  float* dmean;     // [2][pitch]
  int32_t* touch;   // [n]
};

struct AdamArgs {
  float* params;
  const float* grads;
  float* m;
  float* v;
  const float* dmean;
  const int32_t* touch;
  double* stat_norm;
  int32_t* stat_count;
  int64_t pitch, n;
  float lr[5];
  float b1, b2, omb1, omb2, inv_bc1, inv_bc2, eps;
  float ls_lo, ls_hi;
  int accumulate_stats;
};

// Optional per-stage CUDA-event timer (profiling mode of dsg_train).
// Marks: 0 start, 1 preprocess, 2 depth sort, 3 scan+duplicate, 4 tile
// sort+ranges, 5 blend fwd, 6 loss, 7 blend bwd, 8 chain, 9 adam.
struct StageTimer {
  static constexpr int kStages = 9;
  cudaEvent_t ev[kStages + 1] = {};
  bool on = false;
  void mark(int i, cudaStream_t st) {
    if (on) DSG_CUDA_CHECK(cudaEventRecord(ev[i], st));
  }
};

// Sub-tile masks from exact per-row coverage (1, default) or the rect only.
extern std::atomic<int> g_exact_masks;
void bin_frame(Frame& f, const float* params, int64_t pitch, int64_t n, const CamDev& cam,
               const RenderDev& rd, cudaStream_t st, StageTimer* timer = nullptr);
// per tile row: splats whose projected centre falls in it (band balancing)
void center_row_hist_dev(const float* params, int64_t pitch, int64_t n, const CamDev& cam,
                         uint32_t* hist, cudaStream_t st);
void blend_forward(Frame& f, const float* params, int64_t pitch, const CamDev& cam,
                   const RenderDev& rd, cudaStream_t st);
void blend_backward(Frame& f, const float* params, int64_t pitch, const CamDev& cam,
                    const RenderDev& rd, cudaStream_t st);
void chain_3d(const ChainArgs& a, cudaStream_t st);
void adam_update(const AdamArgs& a, cudaStream_t st);
// K7 + K9 in one launch (the training step): gradients never reach HBM;
// a.grads / dmean / touch are not written.
void chain_adam(const ChainArgs& a, const AdamArgs& ad, cudaStream_t st);
// Masked L1 + D-SSIM on f.rgb vs (gt, mask); writes f.dL and the loss into
// `out` (default f.loss_out[0]; device). gt planar fp32 [3][h*w], mask u8 [h*w].
// K11: stamp render_mask discs of `radius` px into a zeroed byte mask.
void render_mask_dev(const double* pts, int64_t n, const CamDev& cam, double radius,
                     uint8_t* mask, cudaStream_t st);
// knn_mean_distances (seed.hpp:16-35): exact grid search; host_pts is the
// host copy of pts (bounds), out on device.
void knn_mean_dev(const double* host_pts, const double* pts, int64_t n, int k, double* out,
                  SortScratch& ss, cudaStream_t st);
// seed_gaussians / ground_truth_model params (seed.hpp:49-94): log-scale from
// scale[i] (or fixed_ls when scale is null), identity rotation.
void seed_params_dev(const double* pts, const double* colors, const double* scale, int64_t n,
                     double fixed_ls, double opacity_logit, float* params, int64_t pitch,
                     cudaStream_t st);
// partition_cloud (partition.hpp:42-104) on the device; lists in index order.
struct PartitionResult {
  int axis = 0;
  std::vector<double> cut_lo, cut_hi, box;  // box: [k][lo xyz, hi xyz]
  std::vector<std::vector<uint32_t>> owned, ghost;
};
PartitionResult partition_dev(const double* host_pts, int64_t n, int nparts, double margin,
                              SortScratch& ss, ScanScratch& sc, cudaStream_t st);
// merge_models keep rule (partition.hpp:120): splats whose mu[axis] lies in
// [cut_lo, cut_hi) are kept, in index order, into a planar dst at dst_off.
// Several partitions at once: merge_trim_count flags and scans all of them
// and reads the counts back with one synchronize; merge_trim_scatter then
// writes partition k's survivors. The flags and prefix sums stay in `ms`
// between the two calls (no allocation once warm).
struct MergeScratch {
  DevBuf<uint32_t> flag, pos, cnt;
  std::vector<int64_t> base;
  std::deque<DevBuf<float>> dense;  // merge exchange: each local partition's survivors, planar
};
struct MergeSrc {
  const float* params;
  int64_t pitch, n;
  double cut_lo, cut_hi;
};
void merge_trim_count(const MergeSrc* src, int np, int axis, MergeScratch& ms, ScanScratch& sc,
                      cudaStream_t st, int64_t* counts);
void merge_trim_scatter(const MergeSrc& src, int k, MergeScratch& ms, float* dst, int64_t dpitch,
                        int64_t dst_off, cudaStream_t st);
// densify_and_prune + AdamState::remap on the device (densify.cu). `spare`
// provides the output storage and receives the old one; rng_state is the
// persistent splitmix64 state of the run's densify Rng (advanced in place).
struct DensifyResult {
  int64_t before = 0, after = 0, splits = 0;
};
// Per-context scratch of densify_dev (classes and three flag scans).
struct DensifyScratch {
  DevBuf<uint8_t> cls;
  DevBuf<uint32_t> cm, ca, cs;
  DevBuf<int> box;
};
DensifyResult densify_dev(ModelDev& m, ModelDev& spare, DensifyScratch& ds, double prune_opacity,
                          double grad_thr,
                          double split_thr_cfg, uint64_t& rng_state, ScanScratch& sc,
                          cudaStream_t st);

// NCCL exchange (comm.cu): ghost-trim merge all-gather, band gather.
extern const char* g_merge_path;  // last merge exchange: "peer" or "nccl"
void nccl_unique_id(uint8_t out[128]);
void* nccl_comm_init(const uint8_t id[128], int nranks, int rank);
void nccl_comm_destroy(void* comm);
void* nccl_comm_split_default(void* comm, int rank);
double bench_allgather_dev(void* comm, int nranks, int64_t bytes, int reps, cudaStream_t st);
int64_t merge_allgather_dev(void* comm, int nranks, int rank, const ModelDev* const* locals,
                            int nlocal, int axis, const double* cut_lo, const double* cut_hi,
                            ModelDev& merged, ScanScratch& sc, MergeScratch& ms, cudaStream_t st,
                            float* wire_ms = nullptr, int64_t* max_iteration = nullptr);
void gather_bands_dev(void* comm, int nranks, int rank, float* rgb, int width, int height,
                      const std::vector<int>& row0, const std::vector<int>& row1, cudaStream_t st);
void masked_loss_dev(Frame& f, const float* gt, const uint8_t* mask, int width, int height,
                     double lambda, cudaStream_t st, double* out = nullptr);

// sum of n_contrib of the last forward and the termination fix-ups (host values)
void frame_work_dev(Frame& f, cudaStream_t st, int64_t* composited, int64_t* fixups,
                    int64_t* changed = nullptr);
// psnr / ssim (metrics.hpp:20-38) of planar fp32 RGB images; out = {psnr, ssim} (device)
void image_metrics_dev(Frame& f, const float* x, const float* y, int width, int height,
                       cudaStream_t st, double* out);

// RT/RM-shaped heightfield clouds on the device (scene.cu); outputs device [n][3]
void heightfield_slice_dev(int64_t n, int64_t s0, int64_t m, uint64_t seed, double span,
                           double amp, double spikes, int nmodes, const double* modes_host,
                           double* pos, double* col, double* nrm, cudaStream_t st);

// float64 PLY (ply_io.hpp:89-221, io.cu)
struct PlyInfo {
  int64_t vertex_count = 0;
  int64_t iteration = 0;
  int origin = -1;
  size_t payload_offset = 0;
};
std::string ply_header(const char* const* props, int nprops, int64_t n, const int64_t* iteration,
                       const int32_t* origin);
void write_file_atomic(const std::string& path, const std::string& head, const char* body,
                       size_t body_bytes);
std::string read_file(const std::string& path);
PlyInfo parse_ply(const std::string& bytes, const char* const* props, int nprops, const char* what);
void splat_ply_payload_dev(const float* params, int64_t pitch, int64_t n, double* out,
                           cudaStream_t st);
void splat_ply_scatter_dev(const double* in, int64_t n, float* params, int64_t pitch,
                           cudaStream_t st);
const char* const* splat_ply_props();
const char* const* cloud_ply_props();

}  // namespace dsg
