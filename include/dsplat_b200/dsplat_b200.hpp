// dsplat_b200.hpp — C++ drop-in for the reference hot path, on the B200.
//
// Same names and signatures as the reference's inline C++ API
// (/root/reference/proj/include/dsplat), in namespace dsplat::b200, over the
// C ABI of libdsg.so (include/dsg.h). The reference's value types
// (SplatModel, Camera, RenderConfig, RenderOutput, Image, TrainView,
// GradientBuffer, TrainConfig, ...) are used unchanged: include this header
// where the reference headers are on the include path, then either call
// dsplat::b200::render(...) or pull the names in with
// `using namespace dsplat::b200;` in place of the CPU implementations.
//
//   reference (file:line)                          drop-in
//   render            render.hpp:160               dsplat::b200::render
//   render_mask       render.hpp:210               dsplat::b200::render_mask
//   masked_loss       loss.hpp:39                  dsplat::b200::masked_loss
//   backward          backward.hpp:184             dsplat::b200::backward
//   AdamState::step   adam.hpp:55                  dsplat::b200::AdamState::step
//   train_partition_full / train_partition
//                     trainer.hpp:140 / :214        dsplat::b200::train_partition_full / ...
//   seed_gaussians / median_nn_spacing / ground_truth_model
//                     seed.hpp:49 / :39 / :78       dsplat::b200::...
//   partition_cloud   partition.hpp:42              dsplat::b200::partition_cloud
//   merge_models      partition.hpp:109             dsplat::b200::merge_models
//     (device-resident models: dsg_merge_models / dsg_merge_allgather)
//   build_orbital_cameras, split_rig, owns: host-side, unchanged from the
//     reference (camera.hpp:75-130, partition.hpp:34-40).
//
// Errors: every failing call throws dsplat::Error with the same ErrorCode and
// what() text ("<Code>: msg") the reference throws (error.hpp:57-61).
// Threading: one Context (device + stream) per thread; Context::current()
// lazily creates one on device 0 for the calling thread.
#pragma once

#include <algorithm>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "dsg.h"
#include "dsplat/error.hpp"
#include "dsplat/loss.hpp"
#include "dsplat/partition.hpp"
#include "dsplat/render.hpp"
#include "dsplat/seed.hpp"
#include "dsplat/trainer.hpp"

namespace dsplat::b200 {

// Throws dsplat::Error for a non-zero dsg status.
inline void check(int rc) {
  if (rc == 0) return;
  std::string what = dsg_last_error();
  std::string msg = what;
  auto p = what.find(": ");
  if (p != std::string::npos) msg = what.substr(p + 2);
  throw Error(static_cast<ErrorCode>(rc - 1), msg);
}

class Context {
 public:
  explicit Context(int device = 0) { check(dsg_ctx_create(device, &h_)); }
  ~Context() { dsg_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  dsg_ctx get() const { return h_; }
  static Context& current() {
    thread_local std::unique_ptr<Context> ctx;
    if (!ctx) ctx = std::make_unique<Context>(0);
    return *ctx;
  }

 private:
  dsg_ctx h_ = nullptr;
};

namespace detail {

inline std::vector<double> params_of(const SplatModel& m) {
  std::vector<double> p(14 * m.size());
  for (size_t i = 0; i < m.size(); ++i) {
    const Gaussian3D& g = m.gaussians[i];
    double* q = p.data() + 14 * i;
    q[0] = g.mu.x; q[1] = g.mu.y; q[2] = g.mu.z;
    q[3] = g.log_scale.x; q[4] = g.log_scale.y; q[5] = g.log_scale.z;
    q[6] = g.rot.w; q[7] = g.rot.x; q[8] = g.rot.y; q[9] = g.rot.z;
    q[10] = g.opacity_logit;
    q[11] = g.color.x; q[12] = g.color.y; q[13] = g.color.z;
  }
  return p;
}

inline void params_to(const std::vector<double>& p, SplatModel& m) {
  m.gaussians.resize(p.size() / 14);
  for (size_t i = 0; i < m.size(); ++i) {
    Gaussian3D& g = m.gaussians[i];
    const double* q = p.data() + 14 * i;
    g.mu = {q[0], q[1], q[2]};
    g.log_scale = {q[3], q[4], q[5]};
    g.rot = {q[6], q[7], q[8], q[9]};
    g.opacity_logit = q[10];
    g.color = {q[11], q[12], q[13]};
  }
}

inline dsg_camera cam_of(const Camera& c) {
  dsg_camera d{};
  d.position[0] = c.position.x; d.position[1] = c.position.y; d.position[2] = c.position.z;
  d.target[0] = c.target.x; d.target[1] = c.target.y; d.target[2] = c.target.z;
  d.up[0] = c.up.x; d.up[1] = c.up.y; d.up[2] = c.up.z;
  d.fov_y = c.fov_y;
  d.width = c.width;
  d.height = c.height;
  d.near_plane = c.near;
  d.far_plane = c.far;
  return d;
}

inline dsg_render_config cfg_of(const RenderConfig& r) {
  dsg_render_config d{};
  d.tile_size = r.tile_size;
  d.alpha_cutoff = r.alpha_cutoff;
  d.sigma_cutoff = r.sigma_cutoff;
  d.background[0] = r.background.x;
  d.background[1] = r.background.y;
  d.background[2] = r.background.z;
  d.transmittance_floor = r.transmittance_floor;
  return d;
}

inline dsg_train_config train_of(const TrainConfig& c) {
  dsg_train_config t{};
  t.iterations = c.iterations;
  t.lr_mu = c.lr_mu;
  t.lr_mu_decay = c.lr_mu_decay;
  t.lr_scale = c.lr_scale;
  t.lr_rot = c.lr_rot;
  t.lr_opacity = c.lr_opacity;
  t.lr_color = c.lr_color;
  t.loss_lambda = c.loss_lambda;
  t.densify_interval = c.densify_interval;
  t.densify_grad_threshold = c.densify_grad_threshold;
  t.prune_opacity = c.prune_opacity;
  t.densify_stop_fraction = c.densify_stop_fraction;
  t.split_scale_threshold = c.split_scale_threshold;
  t.checkpoint_interval = c.checkpoint_interval;
  t.seed = c.seed;
  t.render = cfg_of(c.render);
  t.adam = {c.adam.beta1, c.adam.beta2, c.adam.epsilon};
  return t;
}

// A device copy of a host SplatModel for the duration of one call.
struct DeviceModel {
  dsg_model h = nullptr;
  explicit DeviceModel(const SplatModel& m, Context& ctx) {
    check(dsg_model_create(ctx.get(), &h));
    auto p = params_of(m);
    check(dsg_model_upload(ctx.get(), h, p.data(), static_cast<int64_t>(m.size()), m.iteration,
                           m.origin_partition.value_or(-1)));
  }
  ~DeviceModel() { dsg_model_destroy(h); }
};

}  // namespace detail

// render (render.hpp:160-205).
inline RenderOutput render(const SplatModel& model, const Camera& cam, const RenderConfig& cfg) {
  Context& ctx = Context::current();
  detail::DeviceModel dm(model, ctx);
  RenderOutput out;
  out.color = Image(cam.width, cam.height, 3);
  out.alpha = Image(cam.width, cam.height, 1);
  out.per_pixel_contributor_count.assign(static_cast<size_t>(cam.width) * cam.height, 0);
  out.splat_order.assign(model.size(), 0);
  dsg_camera c = detail::cam_of(cam);
  dsg_render_config r = detail::cfg_of(cfg);
  int64_t n_order = 0, it = 0;
  check(dsg_render(ctx.get(), dm.h, &c, &r, out.color.pixels.data(), out.alpha.pixels.data(),
                   out.per_pixel_contributor_count.data(), out.splat_order.data(), &n_order, &it));
  out.splat_order.resize(static_cast<size_t>(n_order));
  out.model_iteration = it;
  return out;
}

// render_mask (render.hpp:210-233).
inline Image render_mask(const std::vector<Vec3>& points, const Camera& cam, double footprint_px,
                         double dilation_px) {
  Context& ctx = Context::current();
  std::vector<double> pts(3 * points.size());
  for (size_t i = 0; i < points.size(); ++i) {
    pts[3 * i] = points[i].x;
    pts[3 * i + 1] = points[i].y;
    pts[3 * i + 2] = points[i].z;
  }
  Image mask(cam.width, cam.height, 1, 0.0);
  dsg_camera c = detail::cam_of(cam);
  check(dsg_render_mask(ctx.get(), pts.data(), static_cast<int64_t>(points.size()), &c,
                        footprint_px, dilation_px, mask.pixels.data()));
  return mask;
}

// masked_loss (loss.hpp:39-73).
inline LossResult masked_loss(const Image& rendered, const TrainView& view, double loss_lambda) {
  view.validate();
  rendered.require_same_shape(view.ground_truth);
  LossResult r;
  r.dL_dpixels = Image(rendered.width, rendered.height, 3, 0.0);
  check(dsg_masked_loss(Context::current().get(), rendered.pixels.data(),
                        view.ground_truth.pixels.data(), view.mask.pixels.data(), rendered.width,
                        rendered.height, loss_lambda, &r.loss, r.dL_dpixels.pixels.data()));
  return r;
}

// backward (backward.hpp:184-332).
inline GradientBuffer backward(const SplatModel& model, const Camera& cam, const RenderConfig& cfg,
                               const RenderOutput& output, const Image& dL_dpixels,
                               int shards = 1) {
  if (output.model_iteration != model.iteration)
    throw Error(ErrorCode::StaleForward, "render output is from a different model iteration");
  if (dL_dpixels.width != cam.width || dL_dpixels.height != cam.height ||
      dL_dpixels.channels != 3)
    throw Error(ErrorCode::DimensionMismatch, "dL_dpixels must be RGB at camera resolution");
  Context& ctx = Context::current();
  detail::DeviceModel dm(model, ctx);
  const size_t n = model.size();
  std::vector<double> g(14 * n), dm2(2 * n);
  GradientBuffer out(n);
  dsg_camera c = detail::cam_of(cam);
  dsg_render_config r = detail::cfg_of(cfg);
  check(dsg_backward(ctx.get(), dm.h, &c, &r, output.model_iteration, dL_dpixels.pixels.data(),
                     shards, g.data(), dm2.data(), out.touch_count.data()));
  for (size_t i = 0; i < n; ++i) {
    const double* q = g.data() + 14 * i;
    out.d_mu[i] = {q[0], q[1], q[2]};
    out.d_log_scale[i] = {q[3], q[4], q[5]};
    out.d_rot[i] = {q[6], q[7], q[8], q[9]};
    out.d_opacity_logit[i] = q[10];
    out.d_color[i] = {q[11], q[12], q[13]};
    out.d_mean2d[i] = {dm2[2 * i], dm2[2 * i + 1]};
  }
  return out;
}

// AdamState (adam.hpp:19-119): moments live on the device with a private
// device copy of the model being optimised. resize / remap / serialize keep
// the reference's semantics: moments set on the host (remap gathers them,
// resize zeroes them) are installed on the device before the next step.
class AdamState {
 public:
  static constexpr int kScalars = 14;
  explicit AdamState(size_t n = 0) { resize(n); }
  ~AdamState() {
    if (h_) dsg_model_destroy(h_);
  }
  AdamState(const AdamState&) = delete;
  AdamState& operator=(const AdamState&) = delete;
  size_t size() const { return n_; }
  int64_t step_count() const { return step_; }
  using GroupRates = dsplat::AdamState::GroupRates;

  // adam.hpp:26-29: n zeroed moments (the step count is kept)
  void resize(size_t n) {
    n_ = n;
    pm_.assign(n * kScalars, 0.0);
    pv_.assign(n * kScalars, 0.0);
    pending_ = true;
  }

  // adam.hpp:36-49: entry j inherits the moments of source[j] (-1 = fresh)
  void remap(const std::vector<int32_t>& source) {
    std::vector<double> m, v;
    moments(m, v);
    std::vector<double> nm(source.size() * kScalars, 0.0), nv(source.size() * kScalars, 0.0);
    for (size_t j = 0; j < source.size(); ++j) {
      if (source[j] < 0) continue;
      const size_t src = static_cast<size_t>(source[j]);
      std::copy_n(m.begin() + src * kScalars, kScalars, nm.begin() + j * kScalars);
      std::copy_n(v.begin() + src * kScalars, kScalars, nv.begin() + j * kScalars);
    }
    n_ = source.size();
    pm_ = std::move(nm);
    pv_ = std::move(nv);
    pending_ = true;
  }

  // adam.hpp:103-112: [step, size, m..., v...]
  std::vector<double> serialize() const {
    std::vector<double> m, v;
    moments(m, v);
    std::vector<double> out;
    out.reserve(2 + m.size() + v.size());
    out.push_back(static_cast<double>(step_));
    out.push_back(static_cast<double>(n_));
    out.insert(out.end(), m.begin(), m.end());
    out.insert(out.end(), v.begin(), v.end());
    return out;
  }

  // adam.hpp:55-101. Parameters whose device update is zero (no gradient
  // yet) keep their exact fp64 value; updated ones come back as the device
  // computed them (fp32).
  void step(SplatModel& model, const GradientBuffer& grads, const GroupRates& lr,
            const AdamConfig& cfg = {}) {
    Context& ctx = Context::current();
    auto p = detail::params_of(model);
    const int64_t n = static_cast<int64_t>(model.size());
    if (model.size() != n_) resize(model.size());
    if (!h_) check(dsg_model_create(ctx.get(), &h_));
    if (dev_n_ != n) {
      check(dsg_model_upload(ctx.get(), h_, p.data(), n, model.iteration, -1));
      dev_n_ = n;
      pending_ = true;  // upload zeroed the device moments
    } else {
      check(dsg_model_set_params(ctx.get(), h_, p.data(), n, model.iteration));
    }
    if (pending_) {
      check(dsg_model_adam_restore(ctx.get(), h_, pm_.empty() ? nullptr : pm_.data(),
                                   pv_.empty() ? nullptr : pv_.data(), n, step_));
      pending_ = false;
    }
    std::vector<double> g(14 * model.size());
    for (size_t i = 0; i < model.size(); ++i) {
      double* q = g.data() + 14 * i;
      q[0] = grads.d_mu[i].x; q[1] = grads.d_mu[i].y; q[2] = grads.d_mu[i].z;
      q[3] = grads.d_log_scale[i].x; q[4] = grads.d_log_scale[i].y; q[5] = grads.d_log_scale[i].z;
      q[6] = grads.d_rot[i].w; q[7] = grads.d_rot[i].x; q[8] = grads.d_rot[i].y;
      q[9] = grads.d_rot[i].z;
      q[10] = grads.d_opacity_logit[i];
      q[11] = grads.d_color[i].x; q[12] = grads.d_color[i].y; q[13] = grads.d_color[i].z;
    }
    dsg_group_rates r{lr.mu, lr.log_scale, lr.rot, lr.opacity, lr.color};
    dsg_adam_config a{cfg.beta1, cfg.beta2, cfg.epsilon};
    check(dsg_adam_step(ctx.get(), h_, g.data(), &r, &a));
    ++step_;
    std::vector<double> out(p.size());
    int64_t nn = 0, it = 0;
    int32_t op = -1;
    check(dsg_model_download(ctx.get(), h_, out.data(), n, &nn, &it, &op));
    for (size_t k = 0; k < p.size(); ++k)
      if (out[k] != static_cast<double>(static_cast<float>(p[k]))) p[k] = out[k];
    detail::params_to(p, model);
  }

  // A host-only snapshot (checkpoints): moments and step, no device state.
  static std::unique_ptr<AdamState> snapshot(std::vector<double> m, std::vector<double> v,
                                             int64_t step) {
    auto s = std::make_unique<AdamState>(0);
    s->n_ = m.size() / kScalars;
    s->pm_ = std::move(m);
    s->pv_ = std::move(v);
    s->step_ = step;
    s->pending_ = true;
    return s;
  }

 private:
  void moments(std::vector<double>& m, std::vector<double>& v) const {
    if (pending_ || !h_) {
      m = pm_;
      v = pv_;
      m.resize(n_ * kScalars, 0.0);
      v.resize(n_ * kScalars, 0.0);
      return;
    }
    m.assign(n_ * kScalars, 0.0);
    v.assign(n_ * kScalars, 0.0);
    int64_t st = 0;
    check(dsg_model_adam_state(Context::current().get(), h_, m.data(), v.data(), &st));
  }
  dsg_model h_ = nullptr;
  size_t n_ = 0;
  int64_t dev_n_ = -1;
  int64_t step_ = 0;
  std::vector<double> pm_, pv_;
  bool pending_ = false;
};

// CheckpointSink (trainer.hpp:119-120) with the drop-in's AdamState, whose
// serialize() gives the reference's payload (runtime.hpp:262-275 writes it
// to the .adam sidecar). Reference callers that name the type in the lambda
// parameter switch `const AdamState&` to `const auto&`.
using CheckpointSink =
    std::function<void(const SplatModel&, const AdamState&, int64_t iteration, double loss)>;

// train_partition_full (trainer.hpp:140-211): the whole loop on the device.
inline TrainResult train_partition_full(const SplatModel& input,
                                        const std::vector<TrainView>& views,
                                        const TrainConfig& cfg, int shards = 1,
                                        const CheckpointSink& checkpoint = nullptr,
                                        const ProgressSink& progress = nullptr) {
  cfg.validate();
  if (views.empty()) throw Error(ErrorCode::NoViews, "training requires at least one view");
  if (shards < 1) throw Error(ErrorCode::InvalidArgument, "shards must be >= 1");
  for (const auto& v : views) v.validate();
  Context& ctx = Context::current();
  TrainResult result;
  result.model = input;
  result.size_before_densify = input.size();
  result.size_after_densify = input.size();
  if (cfg.iterations == 0) return result;
  detail::DeviceModel dm(input, ctx);
  // the views stay in the caller's TrainView images: dsg_train streams only
  // the scheduled ones, converting each on the host into a pinned slot while
  // the previous step runs
  std::vector<dsg_camera> cams;
  std::vector<const double*> gts, masks;
  for (const auto& v : views) {
    cams.push_back(detail::cam_of(v.cam));
    gts.push_back(v.ground_truth.pixels.data());
    masks.push_back(v.mask.pixels.data());
  }
  dsg_views dv = nullptr;
  check(dsg_views_create_host_ref(ctx.get(), cams.data(), gts.data(), masks.data(),
                                  static_cast<int32_t>(views.size()), &dv));
  std::unique_ptr<dsg_views_s, int (*)(dsg_views)> guard(dv, dsg_views_destroy);
  dsg_train_config tc = detail::train_of(cfg);
  struct Ctx {
    const ProgressSink* p;
    const CheckpointSink* c;
    const SplatModel* input;
    dsg_ctx ctx;
  } pc{&progress, &checkpoint, &input, ctx.get()};
  auto cb = [](int64_t it, double loss, void* u) { (*static_cast<Ctx*>(u)->p)(it, loss); };
  // checkpoint: the model and its moments as the reference hands them over
  auto ck = [](int64_t iter, double loss, dsg_model model, void* u) {
    Ctx& c = *static_cast<Ctx*>(u);
    int64_t n = 0, it = 0, steps = 0;
    check(dsg_model_info(model, &n, &it, &steps));
    std::vector<double> p(14 * static_cast<size_t>(n)), m(p.size()), v(p.size());
    int32_t op = -1;
    check(dsg_model_download(c.ctx, model, p.data(), n, &n, &it, &op));
    check(dsg_model_adam_state(c.ctx, model, m.data(), v.data(), &steps));
    SplatModel snap;
    snap.origin_partition = c.input->origin_partition;
    detail::params_to(p, snap);
    snap.iteration = it;
    auto adam = AdamState::snapshot(std::move(m), std::move(v), steps);
    (*c.c)(snap, *adam, iter, loss);
  };
  check(dsg_train_checkpointed(ctx.get(), dm.h, dv, &tc, shards, progress ? +cb : nullptr, &pc,
                               checkpoint ? +ck : nullptr, &pc, &result.final_loss, nullptr));
  // densify/prune may have resized the model on the device
  int64_t n = 0, it = 0, adam_steps = 0;
  check(dsg_model_info(dm.h, &n, &it, &adam_steps));
  std::vector<double> p(14 * static_cast<size_t>(n));
  int32_t op = -1;
  check(dsg_model_download(ctx.get(), dm.h, p.data(), n, &n, &it, &op));
  detail::params_to(p, result.model);
  result.model.iteration = it;
  result.size_after_densify = result.model.size();
  return result;
}

// train_partition (trainer.hpp:214-217).
inline SplatModel train_partition(const SplatModel& model, const std::vector<TrainView>& views,
                                  const TrainConfig& cfg, int shards = 1) {
  return b200::train_partition_full(model, views, cfg, shards).model;
}

// median_nn_spacing (seed.hpp:39-45) with the exact grid k-NN.
inline double median_nn_spacing(const PointCloud& pc) {
  if (pc.empty()) throw Error(ErrorCode::EmptyCloud, "empty point cloud");
  auto pos = pc.positions();
  std::vector<double> pts(3 * pos.size());
  for (size_t i = 0; i < pos.size(); ++i) {
    pts[3 * i] = pos[i].x;
    pts[3 * i + 1] = pos[i].y;
    pts[3 * i + 2] = pos[i].z;
  }
  double out = 0.0;
  check(dsg_median_nn_spacing(Context::current().get(), pts.data(),
                              static_cast<int64_t>(pos.size()), &out));
  return out;
}

// knn_mean_distances (seed.hpp:16-35).
inline std::vector<double> knn_mean_distances(const PointCloud& pc, int k) {
  std::vector<double> pts(3 * pc.size()), out(pc.size());
  for (size_t i = 0; i < pc.size(); ++i) {
    pts[3 * i] = pc.points[i].position.x;
    pts[3 * i + 1] = pc.points[i].position.y;
    pts[3 * i + 2] = pc.points[i].position.z;
  }
  if (!pc.empty())
    check(dsg_knn_mean(Context::current().get(), pts.data(), static_cast<int64_t>(pc.size()), k,
                       out.data()));
  return out;
}

namespace detail {
inline void cloud_arrays(const PointCloud& pc, std::vector<double>& pts, std::vector<double>& col) {
  pts.resize(3 * pc.size());
  col.resize(3 * pc.size());
  for (size_t i = 0; i < pc.size(); ++i) {
    const SurfacePoint& p = pc.points[i];
    pts[3 * i] = p.position.x;
    pts[3 * i + 1] = p.position.y;
    pts[3 * i + 2] = p.position.z;
    col[3 * i] = p.color.x;
    col[3 * i + 1] = p.color.y;
    col[3 * i + 2] = p.color.z;
  }
}

inline SplatModel download(Context& ctx, dsg_model h) {
  int64_t n = 0, it = 0, st = 0;
  check(dsg_model_info(h, &n, &it, &st));
  std::vector<double> p(14 * static_cast<size_t>(n));
  int32_t op = -1;
  check(dsg_model_download(ctx.get(), h, p.data(), n, &n, &it, &op));
  SplatModel m;
  params_to(p, m);
  m.iteration = it;
  if (op >= 0) m.origin_partition = op;
  return m;
}
}  // namespace detail

// seed_gaussians (seed.hpp:49-74): exact fp64 kNN scales, parameters stored
// (and returned) at the device's fp32 precision.
inline SplatModel seed_gaussians(const PointCloud& pc, ScaleRule rule, int k = 3,
                                 double fixed_scale = 0.01) {
  if (pc.empty()) throw Error(ErrorCode::EmptyCloud, "cannot seed from an empty cloud");
  Context& ctx = Context::current();
  std::vector<double> pts, col;
  detail::cloud_arrays(pc, pts, col);
  dsg_model h = nullptr;
  check(dsg_model_create(ctx.get(), &h));
  std::unique_ptr<dsg_model_s, int (*)(dsg_model)> guard(h, dsg_model_destroy);
  check(dsg_seed_gaussians(ctx.get(), pts.data(), col.data(), static_cast<int64_t>(pc.size()),
                           rule == ScaleRule::Knn ? 0 : 1, k, fixed_scale, h));
  return detail::download(ctx, h);
}

// ground_truth_model (seed.hpp:78-94), fp32 parameters as above.
inline SplatModel ground_truth_model(const PointCloud& pc, double scale_world,
                                     double opacity = 0.97) {
  if (pc.empty()) throw Error(ErrorCode::EmptyCloud, "cannot build ground truth from nothing");
  Context& ctx = Context::current();
  std::vector<double> pts, col;
  detail::cloud_arrays(pc, pts, col);
  dsg_model h = nullptr;
  check(dsg_model_create(ctx.get(), &h));
  std::unique_ptr<dsg_model_s, int (*)(dsg_model)> guard(h, dsg_model_destroy);
  check(dsg_ground_truth_model(ctx.get(), pts.data(), col.data(), static_cast<int64_t>(pc.size()),
                               scale_world, opacity, h));
  return detail::download(ctx, h);
}

// merge_models (partition.hpp:109-126) on the device. The device holds
// parameters as fp32, so the result equals the reference's for the fp32
// models training produces (ownership is tested on the stored mu against the
// fp64 cuts, exactly as `owns`).
inline SplatModel merge_models(const std::vector<SplatModel>& models,
                               const std::vector<Partition>& partitions) {
  if (models.size() != partitions.size())
    throw Error(ErrorCode::MismatchedCounts, "one model per partition required");
  for (size_t k = 0; k < models.size(); ++k) {
    if (!models[k].origin_partition.has_value())
      throw Error(ErrorCode::MismatchedCounts, "model missing origin partition id");
    if (*models[k].origin_partition != partitions[k].id)
      throw Error(ErrorCode::MismatchedCounts, "model/partition id mismatch");
  }
  Context& ctx = Context::current();
  std::vector<std::unique_ptr<detail::DeviceModel>> dms;
  std::vector<dsg_model> hs;
  std::vector<double> lo, hi;
  for (size_t k = 0; k < models.size(); ++k) {
    dms.push_back(std::make_unique<detail::DeviceModel>(models[k], ctx));
    hs.push_back(dms.back()->h);
    lo.push_back(partitions[k].cut_lo);
    hi.push_back(partitions[k].cut_hi);
  }
  dsg_model out = nullptr;
  check(dsg_model_create(ctx.get(), &out));
  std::unique_ptr<dsg_model_s, int (*)(dsg_model)> guard(out, dsg_model_destroy);
  const int axis = partitions.empty() ? 0 : partitions[0].cut_axis;
  check(dsg_merge_models(ctx.get(), hs.data(), static_cast<int32_t>(hs.size()), axis, lo.data(),
                         hi.data(), out));
  SplatModel m = detail::download(ctx, out);
  m.origin_partition.reset();
  return m;
}

// partition_cloud (partition.hpp:42-104): cuts, owned boxes and ownership /
// ghost lists computed on the device in fp64 (bit-identical to the
// reference); the point subsets are gathered here from the caller's cloud.
inline std::vector<Partition> partition_cloud(const PointCloud& pc, int n, double ghost_margin) {
  const auto pos = pc.positions();
  std::vector<double> pts(3 * pos.size());
  for (size_t i = 0; i < pos.size(); ++i) {
    pts[3 * i] = pos[i].x;
    pts[3 * i + 1] = pos[i].y;
    pts[3 * i + 2] = pos[i].z;
  }
  const size_t k = n > 0 ? static_cast<size_t>(n) : 1;
  int32_t axis = 0;
  std::vector<double> lo(k), hi(k), box(6 * k);
  std::vector<int64_t> oc(k), gc(k);
  dsg_ctx ctx = Context::current().get();
  const int64_t np = static_cast<int64_t>(pos.size());
  check(dsg_partition(ctx, pts.data(), np, n, ghost_margin, &axis, lo.data(), hi.data(), box.data(),
                      oc.data(), gc.data(), nullptr, nullptr, 0));  // size query
  int64_t gtot = 0;
  for (int64_t g : gc) gtot += g;
  const int64_t cap = std::max<int64_t>({np, gtot, 1});
  std::vector<uint32_t> oi(cap), gi(cap);
  check(dsg_partition(ctx, pts.data(), np, n, ghost_margin, &axis, lo.data(), hi.data(), box.data(),
                      oc.data(), gc.data(), oi.data(), gi.data(), cap));
  std::vector<Partition> parts(k);
  size_t o = 0, g = 0;
  for (size_t j = 0; j < k; ++j) {
    Partition& p = parts[j];
    p.id = static_cast<int>(j);
    p.ghost_margin = ghost_margin;
    p.cut_axis = axis;
    p.cut_lo = lo[j];
    p.cut_hi = hi[j];
    p.owned_box.lo = {box[6 * j], box[6 * j + 1], box[6 * j + 2]};
    p.owned_box.hi = {box[6 * j + 3], box[6 * j + 4], box[6 * j + 5]};
    p.owned_indices.assign(oi.begin() + o, oi.begin() + o + oc[j]);
    p.ghost_indices.assign(gi.begin() + g, gi.begin() + g + gc[j]);
    for (uint32_t x : p.owned_indices) p.owned_points.points.push_back(pc.points[x]);
    for (uint32_t x : p.ghost_indices) p.ghost_points.points.push_back(pc.points[x]);
    o += oc[j];
    g += gc[j];
  }
  return parts;
}

}  // namespace dsplat::b200
