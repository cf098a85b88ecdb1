/* dsg.h — C ABI of libdsg.so, the B200-native (sm_100a) drop-in for the
 * reference hot path (arxiv 2509.12138 "dsplat", /root/reference/proj).
 *
 * Plain pointers and sizes only. Host arrays use the reference's own
 * layouts so the C++ wrappers in include/dsplat_b200/ are thin:
 *   model params : AoS [n][14] double, order mu(3) log_scale(3) rot wxyz(4)
 *                  opacity_logit(1) color(3)   (adam.hpp:76-98)
 *   RGB images   : row-major HWC double        (image.hpp:34-38)
 *   masks/alpha  : row-major HW double
 * On the device the model is planar fp32 ([14][capacity]) with its Adam
 * moments, gradients and densification statistics resident in HBM.
 *
 * Every call returns 0 on success, otherwise (dsplat::ErrorCode + 1)
 * (error.hpp:10-31), and dsg_last_error() returns the thread-local
 * "<Code>: msg" text that dsplat::Error::what() would give (error.hpp:57-61).
 * A context owns one CUDA device and stream; handles are not thread-safe.
 * There is no CPU fallback: without a usable sm_100 device every call
 * fails with InvalidArgument.
 */
#ifndef DSG_H
#define DSG_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSG_ABI_VERSION 1

typedef struct dsg_ctx_s* dsg_ctx;
typedef struct dsg_model_s* dsg_model;
typedef struct dsg_views_s* dsg_views;

/* dsplat::Camera (camera.hpp:16-24). */
typedef struct {
  double position[3];
  double target[3];
  double up[3];
  double fov_y;
  int32_t width;
  int32_t height;
  double near_plane;
  double far_plane;
} dsg_camera;

/* dsplat::RenderConfig (render.hpp:20-25). */
typedef struct {
  int32_t tile_size;
  int32_t _pad;
  double alpha_cutoff;
  double sigma_cutoff;
  double background[3];
  double transmittance_floor;
} dsg_render_config;

/* dsplat::AdamConfig (adam.hpp:11-15). */
typedef struct {
  double beta1, beta2, epsilon;
} dsg_adam_config;

/* dsplat::AdamState::GroupRates (adam.hpp:51-53). */
typedef struct {
  double mu, log_scale, rot, opacity, color;
} dsg_group_rates;

/* dsplat::TrainConfig (trainer.hpp:13-30). */
typedef struct {
  int64_t iterations;
  double lr_mu, lr_mu_decay, lr_scale, lr_rot, lr_opacity, lr_color;
  double loss_lambda;
  int64_t densify_interval;
  double densify_grad_threshold, prune_opacity, densify_stop_fraction;
  double split_scale_threshold;
  int64_t checkpoint_interval;
  uint64_t seed;
  dsg_render_config render;
  dsg_adam_config adam;
} dsg_train_config;

/* ProgressSink (trainer.hpp:122): (steps completed, current loss). */
typedef void (*dsg_progress_fn)(int64_t iteration, double loss, void* user);

const char* dsg_last_error(void);
int32_t dsg_abi_version(void);

/* ---- context / model ---------------------------------------------------- */
int dsg_ctx_create(int32_t device, dsg_ctx* out);
int dsg_ctx_destroy(dsg_ctx ctx);
int dsg_ctx_synchronize(dsg_ctx ctx);

int dsg_model_create(dsg_ctx ctx, dsg_model* out);
int dsg_model_destroy(dsg_model model);
/* Upload a SplatModel (gaussian.hpp:41-54); resets Adam moments and stats. */
int dsg_model_upload(dsg_ctx ctx, dsg_model model, const double* params, int64_t n,
                     int64_t iteration, int32_t origin_partition);
/* Overwrite the parameters of an existing model of the same size, keeping
 * its Adam moments and statistics (host-side AdamState mirrors). */
int dsg_model_set_params(dsg_ctx ctx, dsg_model model, const double* params, int64_t n,
                         int64_t iteration);
int dsg_model_download(dsg_ctx ctx, dsg_model model, double* params, int64_t capacity,
                       int64_t* n, int64_t* iteration, int32_t* origin_partition);
int dsg_model_info(dsg_model model, int64_t* n, int64_t* iteration, int64_t* adam_step);
/* Adam moments m, v as [n][14] doubles (the AdamState::serialize payload
 * order, adam.hpp:104-112) and the step counter. */
int dsg_model_adam_state(dsg_ctx ctx, dsg_model model, double* m, double* v, int64_t* step);

/* Set the Adam moments (same layout as dsg_model_adam_state; NULL = zeros)
 * and step counter of a device model holding n Gaussians — AdamState::resize
 * / remap (adam.hpp:26-49) and checkpoint resume on the drop-in side. */
int dsg_model_adam_restore(dsg_ctx ctx, dsg_model model, const double* m, const double* v,
                           int64_t n, int64_t step);

/* ---- float64 PLY (ply_io.hpp:89-221) --------------------------------------- */
/* write_splat_ply / read_splat_ply of a device model: byte-identical to
 * serialize_splat_ply of the model's values; load resets the optimizer and
 * takes iteration / origin_partition from the header comments. */
int dsg_model_save_ply(dsg_ctx ctx, dsg_model model, const char* path);
int dsg_model_load_ply(dsg_ctx ctx, dsg_model model, const char* path);
/* write_cloud_ply / read_cloud_ply: positions, normals, colors [n][3]
 * (normals/colors may be NULL: zeros on write, skipped on read); load with
 * positions NULL is a size query into *n. */
int dsg_cloud_save_ply(const char* path, const double* positions, const double* normals,
                       const double* colors, int64_t n);
int dsg_cloud_load_ply(const char* path, double* positions, double* normals, double* colors,
                       int64_t capacity, int64_t* n);

/* ---- synthetic inputs ----------------------------------------- */
/* RT/RM-shaped isosurface cloud y = h(x, z) of n points generated on the
 * device (scene.cu): jittered lattice with hash_combine jitter (rng.hpp:17-20),
 * modes [nmodes][5] = (kx, kz, phase_x, phase_z, amplitude), bubble/spike
 * nonlinearity `spikes`, normal_matte colours (marching_cubes.hpp:21-29);
 * outputs [n][3] fp32-exact doubles (any may be NULL). scenes.py restates it. */
int dsg_heightfield_cloud(dsg_ctx ctx, int64_t n, uint64_t seed, double span, double amp,
                          double spikes, int32_t nmodes, const double* modes, double* positions,
                          double* colors, double* normals);

/* ---- evaluation (metrics.hpp:20-38, runtime.hpp:483-492) ---------------------- */
/* psnr (capped at 99) and mean windowed SSIM of two HWC double RGB images. */
int dsg_image_metrics(dsg_ctx ctx, const double* a, const double* b, int32_t width,
                      int32_t height, double* psnr, double* ssim);
/* psnr / ssim of render(model) against render(truth) at cam, on the device. */
int dsg_eval_view(dsg_ctx ctx, dsg_model model, dsg_model truth, const dsg_camera* cam,
                  const dsg_render_config* cfg, double* psnr, double* ssim);

/* ---- render path ---------------------------------------------------------- */
/* render (render.hpp:160-205). Outputs (each may be NULL): rgb [h][w][3],
 * alpha [h][w], n_contrib [h][w], splat_order (capacity n) and its length,
 * model_iteration (RenderOutput::model_iteration). */
int dsg_render(dsg_ctx ctx, dsg_model model, const dsg_camera* cam,
               const dsg_render_config* cfg, double* rgb, double* alpha, int32_t* n_contrib,
               int32_t* splat_order, int64_t* n_order, int64_t* model_iteration);

/* Per-tile compositing lists of the last dsg_render/dsg_bin on ctx, for
 * parity checks against bin_splats (render.hpp:117-135) at tile_size 16:
 * tile_count[tiles], entries (gaussian indices) capacity given. */
int dsg_bin(dsg_ctx ctx, dsg_model model, const dsg_camera* cam, const dsg_render_config* cfg,
            int32_t* tile_count, int32_t* entries, int64_t capacity, int64_t* n_entries);

/* render_mask (render.hpp:210-233): points [n][3]; mask [h][w] in {0,1}. */
int dsg_render_mask(dsg_ctx ctx, const double* points, int64_t n, const dsg_camera* cam,
                    double footprint_px, double dilation_px, double* mask);

/* masked_loss (loss.hpp:39-73) on host images. */
int dsg_masked_loss(dsg_ctx ctx, const double* rendered, const double* ground_truth,
                    const double* mask, int32_t width, int32_t height, double loss_lambda,
                    double* loss, double* dL_dpixels);

/* backward (backward.hpp:184-332). output_iteration is the
 * RenderOutput::model_iteration of the forward the caller holds
 * (StaleForward if it differs from the model's). The device reduction is
 * shard-invariant, so shards (>= 1) only validates. grads [n][14],
 * d_mean2d [n][2] and touch_count [n] (gradient.hpp:12-46) may be NULL. */
int dsg_backward(dsg_ctx ctx, dsg_model model, const dsg_camera* cam,
                 const dsg_render_config* cfg, int64_t output_iteration,
                 const double* dL_dpixels, int32_t shards, double* grads, double* d_mean2d,
                 int32_t* touch_count);

/* AdamState::step (adam.hpp:55-101) with host gradients [n][14] on the
 * model's device-resident moments; increments the step counter. */
int dsg_adam_step(dsg_ctx ctx, dsg_model model, const double* grads,
                  const dsg_group_rates* rates, const dsg_adam_config* adam);

/* ---- seeding (seed.hpp) ---------------------------------------------------- */
/* knn_mean_distances (seed.hpp:16-35): exact grid k-NN, fp64 distances. */
int dsg_knn_mean(dsg_ctx ctx, const double* points, int64_t n, int32_t k, double* out);
/* median_nn_spacing (seed.hpp:39-45). */
int dsg_median_nn_spacing(dsg_ctx ctx, const double* points, int64_t n, double* out);
/* seed_gaussians (seed.hpp:49-74) straight into a device model.
 * rule: 0 = ScaleRule::Knn (k neighbours), 1 = ScaleRule::Fixed. */
int dsg_seed_gaussians(dsg_ctx ctx, const double* points, const double* colors, int64_t n,
                       int32_t rule, int32_t k, double fixed_scale, dsg_model model);
/* ground_truth_model (seed.hpp:78-94) straight into a device model. */
int dsg_ground_truth_model(dsg_ctx ctx, const double* points, const double* colors, int64_t n,
                           double scale, double opacity, dsg_model model);

/* ---- training -------------------------------------------------------------- */
/* Train views (TrainView, loss.hpp:14-26) resident on the device: ground
 * truth [v][h][w][3] and masks [v][h][w] doubles; all views share (w, h). */
int dsg_views_create(dsg_ctx ctx, const dsg_camera* cams, const double* ground_truth,
                     const double* masks, int32_t n_views, dsg_views* out);
/* make_train_view (runtime.hpp:190-199) on the device: ground truth is the
 * render of gt_model, masks are render_mask of points (or all ones). */
int dsg_views_synthesize(dsg_ctx ctx, dsg_model gt_model, const dsg_render_config* cfg,
                         const dsg_camera* cams, int32_t n_views, const double* points,
                         int64_t n_points, int32_t use_masks, double footprint_px,
                         double dilation_px, dsg_views* out);
/* Views left in caller-owned (pinned) host memory, streamed to the device
 * one step at a time by dsg_train (the end-to-end path): gt_planar[v] is
 * [3][h*w] float, masks[v] is [h*w] bytes; entries the schedule never uses
 * may be NULL. The caller keeps the memory alive until dsg_views_destroy. */
int dsg_views_create_host(dsg_ctx ctx, const dsg_camera* cams, const float* const* gt_planar,
                          const uint8_t* const* masks, int32_t n_views, dsg_views* out);
/* Views in the reference's own TrainView layout (loss.hpp:14-26), left in
 * caller memory: ground_truth[v] is an HWC double image [h][w][3], masks[v]
 * an HW double mask [h][w] (pixel trained iff >= 0.5). dsg_train streams the
 * scheduled views only: per step the host worker pool converts the next view
 * to planar fp32 + bytes in a pinned slot and the copy overlaps the current
 * step. Unused entries may be NULL; the memory must outlive the handle. */
int dsg_views_create_host_ref(dsg_ctx ctx, const dsg_camera* cams,
                              const double* const* ground_truth, const double* const* masks,
                              int32_t n_views, dsg_views* out);
int dsg_views_destroy(dsg_views views);
/* The view index used at each of `iterations` steps for a seed
 * (trainer.hpp:157-163, 174). */
int dsg_view_order(uint64_t seed, int32_t n_views, int64_t iterations, int32_t* out);
/* Copy device view v back in the device layout: gt planar [3][h*w] float,
 * mask [h*w] bytes (either may be NULL) — the input of dsg_views_create_host. */
int dsg_views_download_planar(dsg_ctx ctx, dsg_views views, int32_t v, float* gt_planar,
                              uint8_t* mask);
/* Copy view v back (gt [h][w][3], mask [h][w]; either may be NULL). */
int dsg_views_download(dsg_ctx ctx, dsg_views views, int32_t v, double* ground_truth,
                       double* mask);

/* train_partition_full (trainer.hpp:140-211): the whole loop on the device.
 * The model is updated in place (iteration advances). progress may be NULL;
 * loss_trace (capacity iterations) may be NULL. Densification and pruning
 * (trainer.hpp:47-107, 195-202) run on the device; the model may change
 * size (dsg_model_info reports the new count). */
int dsg_train(dsg_ctx ctx, dsg_model model, dsg_views views, const dsg_train_config* cfg,
              int32_t shards, dsg_progress_fn progress, void* user, double* final_loss,
              double* loss_trace);
/* CheckpointSink (trainer.hpp:119-120): called on the host thread every
 * checkpoint_interval steps and once at the end (trainer.hpp:204-209) with
 * the model's iteration and the step's loss; the stream is idle, so the
 * callback may read `model` with dsg_model_download / dsg_model_adam_state. */
typedef void (*dsg_checkpoint_fn)(int64_t iteration, double loss, dsg_model model, void* user);
/* dsg_train with a checkpoint callback (NULL = none). */
int dsg_train_checkpointed(dsg_ctx ctx, dsg_model model, dsg_views views,
                           const dsg_train_config* cfg, int32_t shards, dsg_progress_fn progress,
                           void* user, dsg_checkpoint_fn checkpoint, void* ckpt_user,
                           double* final_loss, double* loss_trace);

/* ---- partition / merge / multi-GPU (partition.hpp) --------------- */
/* partition_cloud (partition.hpp:42-104) on the device: positions [n][3];
 * cut_lo/cut_hi [nparts], owned_box [nparts][6] (lo xyz, hi xyz), per-part
 * counts, and owned/ghost index lists concatenated in partition order
 * (capacity cap each), every list in ascending point index. With
 * owned_idx or ghost_idx NULL only the counts are written (size query). */
int dsg_partition(dsg_ctx ctx, const double* positions, int64_t n, int32_t nparts, double margin,
                  int32_t* axis, double* cut_lo, double* cut_hi, double* owned_box,
                  int64_t* owned_count, int64_t* ghost_count, uint32_t* owned_idx,
                  uint32_t* ghost_idx, int64_t cap);
/* merge_models (partition.hpp:109-126) of device models in one process:
 * keep splats whose mu[axis] is in [cut_lo[k], cut_hi[k]), in (k, index)
 * order; out.iteration = max. */
int dsg_merge_models(dsg_ctx ctx, const dsg_model* models, int32_t nparts, int32_t axis,
                     const double* cut_lo, const double* cut_hi, dsg_model out);
typedef struct dsg_comm_s* dsg_comm;
/* NCCL communicator over the ranks' GPUs (one rank per process/GPU). */
int dsg_comm_unique_id(uint8_t* out128);
int dsg_comm_create(dsg_ctx ctx, const uint8_t* id128, int32_t nranks, int32_t rank,
                    dsg_comm* out);
int dsg_comm_destroy(dsg_comm comm);
/* Distributed merge: trim this rank's partition model to its owned slab,
 * all-gather survivor counts, broadcast survivors so every rank holds the
 * merged model in (partition = rank, index) order. *ms = device time of
 * the survivor exchange (the NCCL broadcast group, 56 B per survivor). */
int dsg_merge_allgather(dsg_ctx ctx, dsg_comm comm, dsg_model local, int32_t axis, double cut_lo,
                        double cut_hi, dsg_model merged, int64_t* n_merged, double* ms);
/* The same with several partitions per rank: locals[j] holds partition
 * k = j * nranks + rank (partition k on GPU k mod N) with its cuts
 * cut_lo[j], cut_hi[j]; the merged model is in partition order on every rank,
 * iteration = max over partitions. */
int dsg_merge_allgather_multi(dsg_ctx ctx, dsg_comm comm, const dsg_model* locals,
                              int32_t nlocal, int32_t axis, const double* cut_lo,
                              const double* cut_hi, dsg_model merged, int64_t* n_merged,
                              double* ms);
/* How the last merge moved the survivors: "nccl" (one NCCL all-gather of
 * packed records per partition round; the default) or, selected with
 * DSG_MERGE_PATH, "pull" / "push" / "copy" (CUDA IPC mappings of the peers'
 * buffers: NVLink reads with an in-kernel transpose, NVLink writes, or
 * copy-engine plane copies); a peer variant falls back to NCCL when IPC is
 * unavailable. */
const char* dsg_merge_exchange(void);
/* Diagnostic: `reps` NCCL all-gathers of `bytes` per rank on the merge
 * exchange communicator (plain device buffers), each bracketed by CUDA
 * events after a rank alignment; *ms = the mean device time per
 * all-gather. Collective over the communicator's ranks. */
int dsg_comm_bench_allgather(dsg_ctx ctx, dsg_comm comm, int64_t bytes, int32_t reps,
                             double* ms);
/* Tile-parallel render (comm may be NULL): rank r bins and blends tile-row
 * band r of the replicated model, the bands cut at the quantiles of the
 * splats' projected centres per tile row (computed identically on every
 * rank); bands are gathered to rank 0, which
 * receives rgb [h][w][3] (may be NULL). *ms = device time incl. the gather. */
int dsg_render_distributed(dsg_ctx ctx, dsg_comm comm, dsg_model model, const dsg_camera* cam,
                           const dsg_render_config* cfg, double* rgb, double* ms);

/* Number of this library's kernel launches so far (process-wide). */
int64_t dsg_launch_count(void);
/* Visible splats and tile duplicates of the last view binned on ctx. */
int dsg_frame_stats(dsg_ctx ctx, int64_t* n_visible, int64_t* n_dup);
/* Work of the last forward on ctx: composited (pixel, splat) pairs (the sum
 * of n_contrib, the blend kernels' work count C), the pixels
 * whose termination was re-decided in fp64, and how many of those the fp32
 * walk had decided differently. Any pointer may be NULL. */
int dsg_frame_work(dsg_ctx ctx, int64_t* composited, int64_t* term_fixups,
                   int64_t* term_changed);
/* Forward-render n cameras `repeats` times back to back on the device;
 * *ms = CUDA-event time (render Mpix/s measurement). */
int dsg_render_timed(dsg_ctx ctx, dsg_model model, const dsg_camera* cams, int32_t n,
                     const dsg_render_config* cfg, int32_t repeats, double* ms);
/* Page-lock caller memory for the end-to-end path (cudaHostRegister). */
int dsg_host_register(void* ptr, int64_t bytes);
int dsg_host_unregister(void* ptr);

/* NVTX range around a region (lets `ncu --nvtx --nvtx-include name/`
 * profile exactly the bench's timed steps). */
int dsg_nvtx_push(const char* name);
int dsg_nvtx_pop(void);

/* Blend sub-tile masks from exact per-row coverage (1, default) or from the
 * effective rect alone (0). Both give identical results; 0 exists so the
 * parity tests can prove that. Process-wide. */
int dsg_set_exact_masks(int32_t enable);

/* Record per-stage CUDA events inside dsg_train (adds one sync per step). */
int dsg_set_profiling(dsg_ctx ctx, int32_t enable);

/* CUDA-event device time (ms) of the last dsg_train call and, when
 * profiling was on, the per-stage totals (9 entries): preprocess, depth
 * sort, scan+duplicate, tile sort+ranges, blend fwd, loss, blend bwd,
 * 3D chain, Adam. */
int dsg_last_timing(dsg_ctx ctx, double* total_ms, double* stage_ms);

#ifdef __cplusplus
}
#endif
#endif
