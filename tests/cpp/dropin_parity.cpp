// Drop-in parity: the reference C++ API (CPU, /root/reference headers) against
// dsplat::b200 (include/dsplat_b200/dsplat_b200.hpp -> libdsg.so on the B200),
// called with the SAME reference types. Exit code = number of failures.
// Built here by tests/cpp/Makefile (needs the reference headers); the binary
// travels to the GPU box and is run by tests/test_cpp_dropin.py.
#include <cmath>
#include <optional>
#include <cstdio>
#include <string>

#include "dsplat/backward.hpp"
#include "dsplat/trainer.hpp"
#include "dsplat_b200/dsplat_b200.hpp"

using namespace dsplat;

static int failures = 0;
#define EXPECT(cond, ...)                      \
  do {                                         \
    if (!(cond)) {                             \
      ++failures;                              \
      std::printf("FAIL %s: ", #cond);         \
      std::printf(__VA_ARGS__);                \
      std::printf("\n");                       \
    }                                          \
  } while (0)

static float f32(double v) { return static_cast<float>(v); }

static SplatModel scene(uint64_t seed, int n, double scale_mul) {
  Rng rng(seed);
  SplatModel m;
  for (int i = 0; i < n; ++i) {
    Gaussian3D g;
    g.mu = {f32(rng.uniform(-0.5, 0.5)), f32(rng.uniform(-0.5, 0.5)), f32(rng.uniform(-0.4, 0.4))};
    double s = rng.uniform(0.08, 0.35) * scale_mul;
    g.log_scale = {f32(std::log(s * rng.uniform(0.6, 1.6))), f32(std::log(s * rng.uniform(0.6, 1.6))),
                   f32(std::log(s * rng.uniform(0.6, 1.6)))};
    Quat q{rng.normal(), rng.normal(), rng.normal(), rng.normal()};
    q = q.normalized();
    g.rot = {f32(q.w), f32(q.x), f32(q.y), f32(q.z)};
    g.opacity_logit = f32(rng.uniform(-1.0, 1.5));
    g.color = {f32(rng.uniform(0.2, 0.8)), f32(rng.uniform(0.2, 0.8)), f32(rng.uniform(0.2, 0.8))};
    m.gaussians.push_back(g);
  }
  return m;
}

static Camera cam(int res) {
  Camera c;
  c.position = {0.2, 0.1, -3};
  c.target = {0, 0, 0};
  c.width = c.height = res;
  c.near = 0.1;
  c.far = 50;
  return c;
}

int main() {
  RenderConfig cfg;
  for (int k = 0; k < 4; ++k) {
    SplatModel m = scene(100 + k, 40 + 30 * k, k == 3 ? 0.2 : 1.0);
    Camera c = cam(48 + 16 * k);
    RenderOutput a = render(m, c, cfg);
    RenderOutput b = b200::render(m, c, cfg);
    double err = 0;
    for (size_t i = 0; i < a.color.pixels.size(); ++i)
      err = std::max(err, std::abs(a.color.pixels[i] - b.color.pixels[i]));
    EXPECT(err <= 1e-3, "render %d max err %g", k, err);
    EXPECT(a.splat_order == b.splat_order, "render %d splat order", k);

    // masked loss + backward
    TrainView v;
    v.cam = c;
    v.ground_truth = render(scene(200 + k, 40, 1.0), c, cfg).color;
    v.mask = Image(c.width, c.height, 1, 1.0);
    LossResult la = masked_loss(a.color, v, 0.2);
    LossResult lb = b200::masked_loss(a.color, v, 0.2);
    EXPECT(std::abs(la.loss - lb.loss) <= 1e-6 * std::abs(la.loss), "loss %d %g vs %g", k, la.loss,
           lb.loss);
    GradientBuffer ga = backward(m, c, cfg, a, la.dL_dpixels);
    GradientBuffer gb = b200::backward(m, c, cfg, b, la.dL_dpixels);
    double scale = 0, gerr = 0;
    for (size_t i = 0; i < m.size(); ++i) {
      scale = std::max(scale, ga.d_mu[i].norm());
      gerr = std::max(gerr, (ga.d_mu[i] - gb.d_mu[i]).norm());
      EXPECT(ga.touch_count[i] == gb.touch_count[i], "touch %d/%zu", k, i);
    }
    EXPECT(gerr <= 1e-3 * scale, "backward %d d_mu err %g scale %g", k, gerr, scale);
  }
  // errors keep the reference's codes and text
  {
    SplatModel m = scene(5, 3, 1.0);
    RenderOutput out = b200::render(m, cam(32), cfg);
    m.iteration += 1;
    try {
      b200::backward(m, cam(32), cfg, out, Image(32, 32, 3));
      EXPECT(false, "StaleForward not thrown");
    } catch (const Error& e) {
      EXPECT(std::string(e.what()).find("StaleForward") == 0, "what() = %s", e.what());
    }
    try {
      b200::train_partition(m, {}, TrainConfig{});
      EXPECT(false, "NoViews not thrown");
    } catch (const Error& e) {
      EXPECT(e.code() == ErrorCode::NoViews, "code");
    }
  }
  // a short training run tracks the reference
  {
    Camera c = cam(40);
    SplatModel init = scene(23, 12, 1.0);
    TrainView v;
    v.cam = c;
    v.ground_truth = render(scene(24, 12, 1.0), c, cfg).color;
    v.mask = Image(40, 40, 1, 1.0);
    TrainConfig tc;
    tc.iterations = 20;
    tc.seed = 9;
    TrainResult ra = train_partition_full(init, {v}, tc);
    TrainResult rb = b200::train_partition_full(init, {v}, tc);
    EXPECT(std::abs(ra.final_loss - rb.final_loss) <= 2e-3 * ra.final_loss, "train loss %g vs %g",
           ra.final_loss, rb.final_loss);
    EXPECT(rb.model.iteration == init.iteration + 20, "iteration %ld", (long)rb.model.iteration);
  }
  // CheckpointSink (trainer.hpp:204-209): same calls, iterations, losses and
  // serialize() payload shape; moments track the reference's
  {
    Camera c = cam(40);
    SplatModel init = scene(31, 10, 1.0);
    init.origin_partition = 2;
    TrainView v;
    v.cam = c;
    v.ground_truth = render(scene(32, 10, 1.0), c, cfg).color;
    v.mask = Image(40, 40, 1, 1.0);
    TrainConfig tc;
    tc.iterations = 12;
    tc.seed = 5;
    tc.checkpoint_interval = 5;
    struct Ck {
      int64_t iter;
      double loss;
      std::vector<double> adam;
      size_t n;
      std::optional<int> origin;
    };
    std::vector<Ck> ca, cb;
    train_partition_full(init, {v}, tc, 1,
                         [&](const SplatModel& m, const AdamState& a, int64_t it, double l) {
                           ca.push_back({it, l, a.serialize(), m.size(), m.origin_partition});
                         });
    b200::train_partition_full(init, {v}, tc, 1,
                               [&](const SplatModel& m, const auto& a, int64_t it, double l) {
                                 cb.push_back({it, l, a.serialize(), m.size(), m.origin_partition});
                               });
    EXPECT(ca.size() == 3 && cb.size() == ca.size(), "checkpoint calls %zu vs %zu", ca.size(),
           cb.size());
    for (size_t k = 0; k < ca.size() && k < cb.size(); ++k) {
      EXPECT(ca[k].iter == cb[k].iter, "checkpoint %zu iteration %ld vs %ld", k, (long)ca[k].iter,
             (long)cb[k].iter);
      EXPECT(std::abs(ca[k].loss - cb[k].loss) <= 2e-3 * ca[k].loss, "checkpoint %zu loss", k);
      EXPECT(ca[k].adam.size() == cb[k].adam.size() && ca[k].adam[0] == cb[k].adam[0] &&
                 ca[k].adam[1] == cb[k].adam[1], "checkpoint %zu adam header", k);
      EXPECT(ca[k].n == cb[k].n && ca[k].origin == cb[k].origin, "checkpoint %zu model", k);
      double vmax = 0, verr = 0;
      const size_t half = (ca[k].adam.size() - 2) / 2;
      for (size_t i = 2 + half; i < ca[k].adam.size() && i < cb[k].adam.size(); ++i) {
        vmax = std::max(vmax, std::abs(ca[k].adam[i]));
        verr = std::max(verr, std::abs(ca[k].adam[i] - cb[k].adam[i]));
      }
      EXPECT(verr <= 0.05 * vmax, "checkpoint %zu second moments %g of %g", k, verr, vmax);
    }
  }
  // AdamState resize / remap / serialize / step (adam.hpp:24-112)
  {
    Camera c = cam(32);
    SplatModel m = scene(61, 6, 1.0);
    RenderOutput o = render(m, c, cfg);
    TrainView v;
    v.cam = c;
    v.ground_truth = render(scene(62, 6, 1.0), c, cfg).color;
    v.mask = Image(32, 32, 1, 1.0);
    GradientBuffer g = backward(m, c, cfg, o, masked_loss(o.color, v, 0.2).dL_dpixels);
    AdamState ra(m.size());
    b200::AdamState rb(m.size());
    SplatModel ma = m, mb = m;
    AdamState::GroupRates lr{1e-3, 5e-3, 1e-3, 5e-2, 5e-3};
    ra.step(ma, g, lr);
    rb.step(mb, g, lr);
    std::vector<int32_t> src{3, -1, 0, 0, 5, -1, 2};
    ra.remap(src);
    rb.remap(src);
    auto sa = ra.serialize(), sb = rb.serialize();
    EXPECT(sa.size() == sb.size() && sa[0] == sb[0] && sa[1] == sb[1], "remap payload header");
    double err = 0, mx = 0;
    for (size_t i = 2; i < sa.size() && i < sb.size(); ++i) {
      err = std::max(err, std::abs(sa[i] - sb[i]) / std::max(std::abs(sa[i]), 1e-30));
      mx = std::max(mx, std::abs(sa[i]));
    }
    EXPECT(err <= 1e-5, "remapped moments rel err %g", err);
    // untouched scalars keep their exact value after a step (zero update)
    SplatModel m7 = m;
    m7.gaussians.push_back(m.gaussians[0]);
    GradientBuffer g7 = g;
    g7.d_mu.push_back({0, 0, 0});
    g7.d_log_scale.push_back({0, 0, 0});
    g7.d_rot.push_back({0, 0, 0, 0});
    g7.d_opacity_logit.push_back(0.0);
    g7.d_color.push_back({0, 0, 0});
    g7.d_mean2d.push_back({0, 0});
    g7.touch_count.push_back(0);
    g7.d_mu[1] = {0, 0, 0};  // entry 1: fresh moments (remap -1) and no gradient
    SplatModel pa = m7, pb = m7;
    pb.gaussians[1].mu.x = 0.1234567890123;  // not fp32-exact; zero update keeps it exact
    pa.gaussians[1].mu.x = pb.gaussians[1].mu.x;
    ra.step(pa, g7, lr);
    rb.step(pb, g7, lr);
    EXPECT(pb.gaussians[1].mu.x == 0.1234567890123 && pa.gaussians[1].mu.x == pb.gaussians[1].mu.x,
           "zero-update scalar changed: %.17g", pb.gaussians[1].mu.x);
    EXPECT(ra.step_count() == rb.step_count() && rb.step_count() == 2, "step count");
    rb.resize(3);
    EXPECT(rb.size() == 3 && rb.serialize().size() == 2 + 2 * 3 * 14, "resize");
  }
  // densification resizes the model on the device; the drop-in returns it whole
  {
    Camera c = cam(32);
    SplatModel init = scene(45, 8, 1.0);
    init.gaussians[0].log_scale = {f32(std::log(0.5)), f32(std::log(0.35)), f32(std::log(0.25))};
    init.gaussians[1].opacity_logit = -9.0;
    TrainView v;
    v.cam = c;
    v.ground_truth = render(scene(46, 8, 1.0), c, cfg).color;
    v.mask = Image(32, 32, 1, 1.0);
    TrainConfig tc;
    tc.iterations = 60;
    tc.seed = 4;
    tc.densify_interval = 10;
    tc.densify_grad_threshold = 1e-5;
    tc.split_scale_threshold = 0.2;
    TrainResult ra = train_partition_full(init, {v}, tc);
    TrainResult rb = b200::train_partition_full(init, {v}, tc);
    EXPECT(ra.model.size() == rb.model.size() && rb.model.size() != init.size(),
           "densified size %zu vs %zu", ra.model.size(), rb.model.size());
    EXPECT(rb.size_after_densify == rb.model.size(), "size_after_densify");
  }
  // partition_cloud: bit-identical cuts, boxes and lists
  {
    Rng rng(77);
    PointCloud pc;
    for (int i = 0; i < 3000; ++i) {
      SurfacePoint p;
      p.position = {rng.uniform(-1, 1), rng.uniform(-0.5, 0.5), rng.uniform(-2, 2)};
      if (i % 17 == 0) p.position.z = 0.25;  // ties on the cut axis
      pc.points.push_back(p);
    }
    for (int n : {1, 3, 8}) {
      auto a = partition_cloud(pc, n, 0.1);
      auto b = b200::partition_cloud(pc, n, 0.1);
      EXPECT(a.size() == b.size(), "partition count");
      for (size_t k = 0; k < a.size() && k < b.size(); ++k) {
        EXPECT(a[k].cut_axis == b[k].cut_axis && a[k].cut_lo == b[k].cut_lo &&
                   a[k].cut_hi == b[k].cut_hi, "cuts %d/%zu", n, k);
        EXPECT(a[k].owned_indices == b[k].owned_indices, "owned %d/%zu", n, k);
        EXPECT(a[k].ghost_indices == b[k].ghost_indices, "ghosts %d/%zu", n, k);
        EXPECT(a[k].owned_box.lo == b[k].owned_box.lo && a[k].owned_box.hi == b[k].owned_box.hi,
               "box %d/%zu", n, k);
        EXPECT(a[k].owned_points.size() == b[k].owned_points.size(), "owned points %d/%zu", n, k);
      }
    }
    try {
      b200::partition_cloud(PointCloud{}, 2, 0.1);
      EXPECT(false, "EmptyCloud not thrown");
    } catch (const Error& e) {
      EXPECT(e.code() == ErrorCode::EmptyCloud, "code %d", (int)e.code());
    }
    // seeds / ground truth: the reference values rounded to fp32
    {
      PointCloud small;
      small.points.assign(pc.points.begin(), pc.points.begin() + 600);
      const SplatModel sa = seed_gaussians(small, ScaleRule::Knn, 3);
      const SplatModel sb = b200::seed_gaussians(small, ScaleRule::Knn, 3);
      const SplatModel ga = ground_truth_model(small, 0.01, 0.97);
      const SplatModel gb = b200::ground_truth_model(small, 0.01, 0.97);
      EXPECT(sa.size() == sb.size() && ga.size() == gb.size(), "seed sizes");
      // relative error within fp32 rounding (device fp64 log may differ from
      // glibc's by an ulp before the fp32 rounding)
      double serr = 0;
      auto rel = [](double a, double b) { return std::abs(a - b) / std::max(std::abs(a), 1e-30); };
      for (size_t i = 0; i < sa.size() && i < sb.size(); ++i) {
        serr = std::max(serr, rel(sa.gaussians[i].log_scale.x, sb.gaussians[i].log_scale.x));
        serr = std::max(serr, rel(sa.gaussians[i].opacity_logit, sb.gaussians[i].opacity_logit));
        serr = std::max(serr, rel(ga.gaussians[i].log_scale.y, gb.gaussians[i].log_scale.y));
        serr = std::max(serr, rel(ga.gaussians[i].mu.z, gb.gaussians[i].mu.z));
      }
      EXPECT(serr <= 2e-7, "seed/gt values differ by %g relative", serr);
    }
    // merge_models on fp32-exact models: identical to the reference
    {
      auto parts = partition_cloud(pc, 3, 0.1);
      std::vector<SplatModel> models;
      for (int k = 0; k < 3; ++k) {
        SplatModel m = scene(300 + k, 200 + 50 * k, 1.0);
        for (auto& g : m.gaussians) {  // spread over the cut axis range
          g.mu.z = f32(g.mu.z * 4.0);
        }
        m.origin_partition = k;
        m.iteration = 10 + k;
        models.push_back(m);
      }
      const SplatModel ma = merge_models(models, parts);
      const SplatModel mb = b200::merge_models(models, parts);
      EXPECT(ma.size() == mb.size(), "merge size %zu vs %zu", ma.size(), mb.size());
      EXPECT(ma.iteration == mb.iteration, "merge iteration");
      bool same = ma.size() == mb.size();
      for (size_t i = 0; same && i < ma.size(); ++i)
        same = ma.gaussians[i].mu == mb.gaussians[i].mu &&
               ma.gaussians[i].opacity_logit == mb.gaussians[i].opacity_logit;
      EXPECT(same, "merged splats differ");
      try {
        models[1].origin_partition = 2;
        b200::merge_models(models, parts);
        EXPECT(false, "MismatchedCounts not thrown");
      } catch (const Error& e) {
        EXPECT(e.code() == ErrorCode::MismatchedCounts, "merge code %d", (int)e.code());
      }
    }
  }
  std::printf("dropin_parity: %d failure(s)\n", failures);
  return failures;
}
