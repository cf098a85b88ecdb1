/* TEST INFRASTRUCTURE ONLY — never linked into the product library.
 *
 * C ABI shared by the two CPU checkers under oracle/:
 *   - liboracle.so        : oracle.cpp, this repo's own fp64 restatement of
 *                           the reference algorithm (proj/include/dsplat/…)
 *   - _ref/libdsplat_ref.so: ref_shim.cpp, the UNMODIFIED reference headers
 *                           (/root/reference/proj/include) compiled here and
 *                           wrapped in the same ABI, used to pin oracle.cpp.
 * Both are loaded by tests/ (and bench.py's cpu_baseline leg) through
 * oracle/__init__.py. Everything is double precision, AoS, in the
 * reference's own layouts:
 *   model params : [n][14]  mu(3) log_scale(3) rot wxyz(4) opacity_logit(1)
 *                  color(3) — the flat order of adam.hpp:76-98
 *   images       : row-major HWC doubles (image.hpp:34-38)
 *   grads        : [n][14] in the same order; d_mean2d [n][2]; touch [n]
 * Return value: 0 on success, else (dsplat::ErrorCode + 1) (error.hpp:10-31);
 * orc_last_error() gives "<Code>: msg" like Error::what() (error.hpp:57-61).
 */
#ifndef DSPLAT_ORC_ABI_H
#define DSPLAT_ORC_ABI_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double position[3];
  double target[3];
  double up[3];
  double fov_y;
  int32_t width;
  int32_t height;
  double near_plane;
  double far_plane;
} orc_camera;

typedef struct {
  int32_t tile_size;
  int32_t _pad;
  double alpha_cutoff;
  double sigma_cutoff;
  double background[3];
  double transmittance_floor;
} orc_render_cfg;

typedef struct {
  int64_t iterations;
  double lr_mu, lr_mu_decay, lr_scale, lr_rot, lr_opacity, lr_color;
  double loss_lambda;
  int64_t densify_interval;
  double densify_grad_threshold, prune_opacity, densify_stop_fraction;
  double split_scale_threshold;
  int64_t checkpoint_interval;
  uint64_t seed;
  orc_render_cfg render;
  double beta1, beta2, epsilon;
} orc_train_cfg;

const char* orc_last_error(void);
const char* orc_impl_name(void);

/* prepare_splats (render.hpp:62-103): projected, culled, depth-sorted list.
 * Outputs have capacity n; *n_out receives the visible count. */
int orc_prepare(const double* params, int64_t n, const orc_camera* cam, const orc_render_cfg* cfg,
                int64_t* n_out, int32_t* index, double* mean2d, double* inv_cov, double* opacity,
                double* depth, int32_t* rect);

/* bin_splats (render.hpp:117-135): per-tile lists of GAUSSIAN indices in
 * compositing order. tile_count[n_tiles]; entries capacity given; returns
 * total entries in *n_entries (InvalidArgument if capacity too small). */
int orc_bin(const double* params, int64_t n, const orc_camera* cam, const orc_render_cfg* cfg,
            int32_t* tile_count, int32_t* entries, int64_t capacity, int64_t* n_entries);

/* render (render.hpp:160-205). splat_order capacity n. */
int orc_render(const double* params, int64_t n, const orc_camera* cam, const orc_render_cfg* cfg,
               double* rgb, double* alpha, int32_t* n_contrib, int32_t* splat_order,
               int64_t* n_order);

/* render_mask (render.hpp:210-233). points [n][3]; mask h*w doubles. */
int orc_render_mask(const double* points, int64_t n, const orc_camera* cam, double footprint_px,
                    double dilation_px, double* mask);

/* masked_loss (loss.hpp:39-73). */
int orc_masked_loss(const double* rendered, const double* gt, const double* mask, int32_t width,
                    int32_t height, double lambda, double* loss, double* dL);

/* ssim (metrics.hpp:33-38) and psnr (metrics.hpp:20-30), for evaluation. */
int orc_ssim(const double* a, const double* b, int32_t width, int32_t height, double* out);
int orc_psnr(const double* a, const double* b, int64_t count, double* out);

/* backward (backward.hpp:184-332). */
int orc_backward(const double* params, int64_t n, int64_t model_iteration,
                 int64_t output_iteration, const orc_camera* cam, const orc_render_cfg* cfg,
                 const double* dL, int32_t shards, double* grads, double* d_mean2d,
                 int32_t* touch);

/* AdamState::step (adam.hpp:55-101). m, v are [n][14]; *step is the
 * optimizer step counter (incremented). rates = {mu, log_scale, rot,
 * opacity, color}; adam = {beta1, beta2, epsilon}. */
int orc_adam_step(double* params, int64_t n, const double* grads, double* m, double* v,
                  int64_t* step, const double* rates, const double* adam);

/* train_partition_full (trainer.hpp:140-211). All views share width/height.
 * params_out capacity cap_out (densification may grow the model). */
int orc_train(const double* params_in, int64_t n, const orc_camera* cams, const double* gts,
              const double* masks, int32_t n_views, const orc_train_cfg* cfg, int32_t shards,
              double* params_out, int64_t cap_out, int64_t* n_out, double* final_loss,
              double* loss_trace);

/* partition_cloud (partition.hpp:42-104). positions [n][3].
 * Outputs: axis, cut_lo[nparts], cut_hi[nparts], owned_box[nparts][6],
 * owned_count/ghost_count [nparts]; owned_idx / ghost_idx concatenated in
 * partition order (capacity cap each). */
int orc_partition(const double* positions, int64_t n, int32_t nparts, double margin,
                  int32_t* axis, double* cut_lo, double* cut_hi, double* owned_box,
                  int64_t* owned_count, int64_t* ghost_count, uint32_t* owned_idx,
                  uint32_t* ghost_idx, int64_t cap);

/* merge_models (partition.hpp:109-126) for already-partitioned models:
 * models concatenated [sum n_k][14]; keep flags returned per input splat. */
int orc_merge(const double* params, const int64_t* counts, int32_t nparts, int32_t axis,
              const double* cut_lo, const double* cut_hi, uint8_t* keep, int64_t* n_kept);

/* build_orbital_cameras (camera.hpp:75-107). out capacity n_az*n_el. */
int orc_orbital_cameras(const double* center, double radius, int32_t n_az, int32_t n_el,
                        int32_t resolution, double fov_y, double max_elevation, orc_camera* out);

/* split_rig (camera.hpp:116-130). train/test index arrays capacity n. */
int orc_split_rig(int64_t n_views, double test_fraction, uint64_t seed, int32_t* train,
                  int64_t* n_train, int32_t* test, int64_t* n_test);

/* knn_mean_distances / median_nn_spacing / seed_gaussians /
 * ground_truth_model (seed.hpp). points [n][3], colors [n][3]. */
int orc_knn_mean(const double* points, int64_t n, int32_t k, double* out);
int orc_median_nn(const double* points, int64_t n, double* out);
int orc_seed_knn(const double* points, const double* colors, int64_t n, int32_t k,
                 double* params);
int orc_gt_model(const double* points, const double* colors, int64_t n, double scale,
                 double opacity, double* params);

/* Rng stream (rng.hpp:8-64): writes count uniform() draws. */
int orc_rng_uniform(uint64_t seed, int64_t count, double* out);

#ifdef __cplusplus
}
#endif
#endif
