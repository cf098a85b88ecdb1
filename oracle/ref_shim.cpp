// TEST INFRASTRUCTURE ONLY. Wraps the UNMODIFIED reference headers
// (/root/reference/proj/include/dsplat, compiled in place by oracle/Makefile
// into oracle/_ref/libdsplat_ref.so) behind the oracle C ABI in orc_abi.h.
// Used to pin oracle.cpp (tests/test_oracle_pin.py), to generate the golden
// fixtures (tests/golden/make_golden.py) and as bench.py's "reference" CPU
// baseline. Nothing in the product library links or loads this.
#include <cstring>
#include <string>

#include "dsplat/backward.hpp"
#include "dsplat/metrics.hpp"
#include "dsplat/partition.hpp"
#include "dsplat/ply_io.hpp"
#include "dsplat/seed.hpp"
#include "dsplat/trainer.hpp"
#include "orc_abi.h"

using namespace dsplat;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = std::string("InvalidArgument: ") + e.what();
    return static_cast<int>(ErrorCode::InvalidArgument) + 1;
  }
}

SplatModel to_model(const double* p, int64_t n) {
  SplatModel m;
  m.gaussians.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    const double* q = p + 14 * i;
    Gaussian3D& g = m.gaussians[static_cast<size_t>(i)];
    g.mu = {q[0], q[1], q[2]};
    g.log_scale = {q[3], q[4], q[5]};
    g.rot = {q[6], q[7], q[8], q[9]};
    g.opacity_logit = q[10];
    g.color = {q[11], q[12], q[13]};
  }
  return m;
}

void from_model(const SplatModel& m, double* p) {
  for (size_t i = 0; i < m.size(); ++i) {
    const Gaussian3D& g = m.gaussians[i];
    double* q = p + 14 * i;
    q[0] = g.mu.x; q[1] = g.mu.y; q[2] = g.mu.z;
    q[3] = g.log_scale.x; q[4] = g.log_scale.y; q[5] = g.log_scale.z;
    q[6] = g.rot.w; q[7] = g.rot.x; q[8] = g.rot.y; q[9] = g.rot.z;
    q[10] = g.opacity_logit;
    q[11] = g.color.x; q[12] = g.color.y; q[13] = g.color.z;
  }
}

Camera to_cam(const orc_camera* c) {
  Camera cam;
  cam.position = {c->position[0], c->position[1], c->position[2]};
  cam.target = {c->target[0], c->target[1], c->target[2]};
  cam.up = {c->up[0], c->up[1], c->up[2]};
  cam.fov_y = c->fov_y;
  cam.width = c->width;
  cam.height = c->height;
  cam.near = c->near_plane;
  cam.far = c->far_plane;
  return cam;
}

void from_cam(const Camera& cam, orc_camera* c) {
  c->position[0] = cam.position.x; c->position[1] = cam.position.y; c->position[2] = cam.position.z;
  c->target[0] = cam.target.x; c->target[1] = cam.target.y; c->target[2] = cam.target.z;
  c->up[0] = cam.up.x; c->up[1] = cam.up.y; c->up[2] = cam.up.z;
  c->fov_y = cam.fov_y;
  c->width = cam.width;
  c->height = cam.height;
  c->near_plane = cam.near;
  c->far_plane = cam.far;
}

RenderConfig to_cfg(const orc_render_cfg* c) {
  RenderConfig r;
  r.tile_size = c->tile_size;
  r.alpha_cutoff = c->alpha_cutoff;
  r.sigma_cutoff = c->sigma_cutoff;
  r.background = {c->background[0], c->background[1], c->background[2]};
  r.transmittance_floor = c->transmittance_floor;
  return r;
}

Image to_image(const double* px, int w, int h, int c) {
  Image img(w, h, c);
  std::memcpy(img.pixels.data(), px, sizeof(double) * img.pixels.size());
  return img;
}

PointCloud to_cloud(const double* pts, const double* colors, int64_t n) {
  PointCloud pc;
  pc.points.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    auto& p = pc.points[static_cast<size_t>(i)];
    p.position = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    if (colors) p.color = {colors[3 * i], colors[3 * i + 1], colors[3 * i + 2]};
    p.normal = {0, 0, 1};
  }
  return pc;
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
const char* orc_impl_name(void) { return "reference"; }

int orc_prepare(const double* params, int64_t n, const orc_camera* cam, const orc_render_cfg* cfg,
                int64_t* n_out, int32_t* index, double* mean2d, double* inv_cov, double* opacity,
                double* depth, int32_t* rect) {
  return guarded([&] {
    SplatModel m = to_model(params, n);
    auto prep = detail::prepare_splats(m, to_cam(cam), to_cfg(cfg));
    *n_out = static_cast<int64_t>(prep.size());
    for (size_t i = 0; i < prep.size(); ++i) {
      const auto& p = prep[i];
      index[i] = p.index;
      mean2d[2 * i] = p.mean2d.x;
      mean2d[2 * i + 1] = p.mean2d.y;
      inv_cov[3 * i] = p.inv_cov2d.xx;
      inv_cov[3 * i + 1] = p.inv_cov2d.xy;
      inv_cov[3 * i + 2] = p.inv_cov2d.yy;
      opacity[i] = p.opacity;
      depth[i] = p.depth;
      rect[4 * i] = p.x0;
      rect[4 * i + 1] = p.x1;
      rect[4 * i + 2] = p.y0;
      rect[4 * i + 3] = p.y1;
    }
  });
}

int orc_bin(const double* params, int64_t n, const orc_camera* cam, const orc_render_cfg* cfg,
            int32_t* tile_count, int32_t* entries, int64_t capacity, int64_t* n_entries) {
  return guarded([&] {
    SplatModel m = to_model(params, n);
    Camera c = to_cam(cam);
    RenderConfig r = to_cfg(cfg);
    auto prep = detail::prepare_splats(m, c, r);
    auto bins = detail::bin_splats(prep, c.width, c.height, r.tile_size);
    int64_t total = 0;
    for (size_t t = 0; t < bins.bins.size(); ++t) {
      tile_count[t] = static_cast<int32_t>(bins.bins[t].size());
      for (int32_t pos : bins.bins[t]) {
        if (total < capacity) entries[total] = prep[static_cast<size_t>(pos)].index;
        ++total;
      }
    }
    *n_entries = total;
    if (total > capacity) throw Error(ErrorCode::InvalidArgument, "entry capacity too small");
  });
}

int orc_render(const double* params, int64_t n, const orc_camera* cam, const orc_render_cfg* cfg,
               double* rgb, double* alpha, int32_t* n_contrib, int32_t* splat_order,
               int64_t* n_order) {
  return guarded([&] {
    SplatModel m = to_model(params, n);
    RenderOutput out = render(m, to_cam(cam), to_cfg(cfg));
    std::memcpy(rgb, out.color.pixels.data(), sizeof(double) * out.color.pixels.size());
    std::memcpy(alpha, out.alpha.pixels.data(), sizeof(double) * out.alpha.pixels.size());
    std::memcpy(n_contrib, out.per_pixel_contributor_count.data(),
                sizeof(int32_t) * out.per_pixel_contributor_count.size());
    *n_order = static_cast<int64_t>(out.splat_order.size());
    if (splat_order)
      std::memcpy(splat_order, out.splat_order.data(), sizeof(int32_t) * out.splat_order.size());
  });
}

int orc_render_mask(const double* points, int64_t n, const orc_camera* cam, double footprint_px,
                    double dilation_px, double* mask) {
  return guarded([&] {
    std::vector<Vec3> pts(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) pts[static_cast<size_t>(i)] = {points[3 * i], points[3 * i + 1], points[3 * i + 2]};
    Image img = render_mask(pts, to_cam(cam), footprint_px, dilation_px);
    std::memcpy(mask, img.pixels.data(), sizeof(double) * img.pixels.size());
  });
}

int orc_masked_loss(const double* rendered, const double* gt, const double* mask, int32_t width,
                    int32_t height, double lambda, double* loss, double* dL) {
  return guarded([&] {
    TrainView view;
    view.cam.width = width;
    view.cam.height = height;
    view.ground_truth = to_image(gt, width, height, 3);
    view.mask = to_image(mask, width, height, 1);
    LossResult r = masked_loss(to_image(rendered, width, height, 3), view, lambda);
    *loss = r.loss;
    std::memcpy(dL, r.dL_dpixels.pixels.data(), sizeof(double) * r.dL_dpixels.pixels.size());
  });
}

int orc_ssim(const double* a, const double* b, int32_t width, int32_t height, double* out) {
  return guarded([&] { *out = ssim(to_image(a, width, height, 3), to_image(b, width, height, 3)); });
}

int orc_psnr(const double* a, const double* b, int64_t count, double* out) {
  return guarded([&] {
    *out = psnr(to_image(a, static_cast<int>(count), 1, 1), to_image(b, static_cast<int>(count), 1, 1));
  });
}

int orc_backward(const double* params, int64_t n, int64_t model_iteration,
                 int64_t output_iteration, const orc_camera* cam, const orc_render_cfg* cfg,
                 const double* dL, int32_t shards, double* grads, double* d_mean2d,
                 int32_t* touch) {
  return guarded([&] {
    SplatModel m = to_model(params, n);
    m.iteration = model_iteration;
    RenderOutput out;
    out.model_iteration = output_iteration;
    Camera c = to_cam(cam);
    GradientBuffer g = backward(m, c, to_cfg(cfg), out, to_image(dL, c.width, c.height, 3), shards);
    for (int64_t i = 0; i < n; ++i) {
      size_t k = static_cast<size_t>(i);
      double* q = grads + 14 * i;
      q[0] = g.d_mu[k].x; q[1] = g.d_mu[k].y; q[2] = g.d_mu[k].z;
      q[3] = g.d_log_scale[k].x; q[4] = g.d_log_scale[k].y; q[5] = g.d_log_scale[k].z;
      q[6] = g.d_rot[k].w; q[7] = g.d_rot[k].x; q[8] = g.d_rot[k].y; q[9] = g.d_rot[k].z;
      q[10] = g.d_opacity_logit[k];
      q[11] = g.d_color[k].x; q[12] = g.d_color[k].y; q[13] = g.d_color[k].z;
      if (d_mean2d) {
        d_mean2d[2 * i] = g.d_mean2d[k].x;
        d_mean2d[2 * i + 1] = g.d_mean2d[k].y;
      }
      if (touch) touch[i] = g.touch_count[k];
    }
  });
}

int orc_adam_step(double* params, int64_t n, const double* grads, double* m, double* v,
                  int64_t* step, const double* rates, const double* adam) {
  // AdamState keeps its moments private (adam.hpp:114-118), so the shim can
  // only drive a fresh optimizer: step 0 with zero moments. Multi-step
  // trajectories are pinned through orc_train instead.
  return guarded([&] {
    for (int64_t i = 0; i < 14 * n; ++i)
      if (m[i] != 0.0 || v[i] != 0.0)
        throw Error(ErrorCode::InvalidArgument, "ref adam shim supports a fresh state only");
    if (*step != 0) throw Error(ErrorCode::InvalidArgument, "ref adam shim supports step 0 only");
    SplatModel model = to_model(params, n);
    GradientBuffer g(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      size_t k = static_cast<size_t>(i);
      const double* q = grads + 14 * i;
      g.d_mu[k] = {q[0], q[1], q[2]};
      g.d_log_scale[k] = {q[3], q[4], q[5]};
      g.d_rot[k] = {q[6], q[7], q[8], q[9]};
      g.d_opacity_logit[k] = q[10];
      g.d_color[k] = {q[11], q[12], q[13]};
    }
    AdamState st(static_cast<size_t>(n));
    AdamConfig ac{adam[0], adam[1], adam[2]};
    st.step(model, g, {rates[0], rates[1], rates[2], rates[3], rates[4]}, ac);
    from_model(model, params);
    auto ser = st.serialize();
    *step = static_cast<int64_t>(ser[0]);
    std::memcpy(m, ser.data() + 2, sizeof(double) * 14 * static_cast<size_t>(n));
    std::memcpy(v, ser.data() + 2 + 14 * n, sizeof(double) * 14 * static_cast<size_t>(n));
  });
}

int orc_train(const double* params_in, int64_t n, const orc_camera* cams, const double* gts,
              const double* masks, int32_t n_views, const orc_train_cfg* cfg, int32_t shards,
              double* params_out, int64_t cap_out, int64_t* n_out, double* final_loss,
              double* loss_trace) {
  return guarded([&] {
    std::vector<TrainView> views(static_cast<size_t>(n_views));
    for (int32_t v = 0; v < n_views; ++v) {
      TrainView& tv = views[static_cast<size_t>(v)];
      tv.cam = to_cam(&cams[v]);
      size_t px = static_cast<size_t>(tv.cam.width) * static_cast<size_t>(tv.cam.height);
      tv.ground_truth = to_image(gts + 3 * px * static_cast<size_t>(v), tv.cam.width, tv.cam.height, 3);
      tv.mask = to_image(masks + px * static_cast<size_t>(v), tv.cam.width, tv.cam.height, 1);
    }
    TrainConfig tc;
    tc.iterations = cfg->iterations;
    tc.lr_mu = cfg->lr_mu;
    tc.lr_mu_decay = cfg->lr_mu_decay;
    tc.lr_scale = cfg->lr_scale;
    tc.lr_rot = cfg->lr_rot;
    tc.lr_opacity = cfg->lr_opacity;
    tc.lr_color = cfg->lr_color;
    tc.loss_lambda = cfg->loss_lambda;
    tc.densify_interval = cfg->densify_interval;
    tc.densify_grad_threshold = cfg->densify_grad_threshold;
    tc.prune_opacity = cfg->prune_opacity;
    tc.densify_stop_fraction = cfg->densify_stop_fraction;
    tc.split_scale_threshold = cfg->split_scale_threshold;
    tc.checkpoint_interval = cfg->checkpoint_interval;
    tc.seed = cfg->seed;
    tc.render = to_cfg(&cfg->render);
    tc.adam = AdamConfig{cfg->beta1, cfg->beta2, cfg->epsilon};
    ProgressSink progress = nullptr;
    if (loss_trace)
      progress = [&](int64_t it, double loss) { loss_trace[it - 1] = loss; };
    TrainResult r = train_partition_full(to_model(params_in, n), views, tc, shards, nullptr, progress);
    if (static_cast<int64_t>(r.model.size()) > cap_out)
      throw Error(ErrorCode::InvalidArgument, "output capacity too small");
    from_model(r.model, params_out);
    *n_out = static_cast<int64_t>(r.model.size());
    *final_loss = r.final_loss;
  });
}

int orc_partition(const double* positions, int64_t n, int32_t nparts, double margin,
                  int32_t* axis, double* cut_lo, double* cut_hi, double* owned_box,
                  int64_t* owned_count, int64_t* ghost_count, uint32_t* owned_idx,
                  uint32_t* ghost_idx, int64_t cap) {
  return guarded([&] {
    PointCloud pc = to_cloud(positions, nullptr, n);
    auto parts = partition_cloud(pc, nparts, margin);
    int64_t oi = 0, gi = 0;
    for (int32_t k = 0; k < nparts; ++k) {
      const Partition& p = parts[static_cast<size_t>(k)];
      *axis = p.cut_axis;
      cut_lo[k] = p.cut_lo;
      cut_hi[k] = p.cut_hi;
      double* b = owned_box + 6 * k;
      b[0] = p.owned_box.lo.x; b[1] = p.owned_box.lo.y; b[2] = p.owned_box.lo.z;
      b[3] = p.owned_box.hi.x; b[4] = p.owned_box.hi.y; b[5] = p.owned_box.hi.z;
      owned_count[k] = static_cast<int64_t>(p.owned_indices.size());
      ghost_count[k] = static_cast<int64_t>(p.ghost_indices.size());
      for (uint32_t x : p.owned_indices) {
        if (oi < cap) owned_idx[oi] = x;
        ++oi;
      }
      for (uint32_t x : p.ghost_indices) {
        if (gi < cap) ghost_idx[gi] = x;
        ++gi;
      }
    }
    if (oi > cap || gi > cap) throw Error(ErrorCode::InvalidArgument, "index capacity too small");
  });
}

int orc_merge(const double* params, const int64_t* counts, int32_t nparts, int32_t axis,
              const double* cut_lo, const double* cut_hi, uint8_t* keep, int64_t* n_kept) {
  return guarded([&] {
    std::vector<SplatModel> models(static_cast<size_t>(nparts));
    std::vector<Partition> parts(static_cast<size_t>(nparts));
    int64_t off = 0;
    for (int32_t k = 0; k < nparts; ++k) {
      models[static_cast<size_t>(k)] = to_model(params + 14 * off, counts[k]);
      models[static_cast<size_t>(k)].origin_partition = k;
      parts[static_cast<size_t>(k)].id = k;
      parts[static_cast<size_t>(k)].cut_axis = axis;
      parts[static_cast<size_t>(k)].cut_lo = cut_lo[k];
      parts[static_cast<size_t>(k)].cut_hi = cut_hi[k];
      off += counts[k];
    }
    SplatModel merged = merge_models(models, parts);
    // Recover keep flags with the reference's own predicate.
    off = 0;
    int64_t kept = 0;
    for (int32_t k = 0; k < nparts; ++k)
      for (int64_t i = 0; i < counts[k]; ++i, ++off) {
        bool o = owns(parts[static_cast<size_t>(k)], models[static_cast<size_t>(k)].gaussians[static_cast<size_t>(i)].mu);
        keep[off] = o ? 1 : 0;
        kept += o ? 1 : 0;
      }
    if (kept != static_cast<int64_t>(merged.size()))
      throw Error(ErrorCode::MismatchedCounts, "merge size mismatch");
    *n_kept = kept;
  });
}

int orc_orbital_cameras(const double* center, double radius, int32_t n_az, int32_t n_el,
                        int32_t resolution, double fov_y, double max_elevation, orc_camera* out) {
  return guarded([&] {
    auto rig = build_orbital_cameras({center[0], center[1], center[2]}, radius, n_az, n_el,
                                     resolution, fov_y, max_elevation);
    for (size_t i = 0; i < rig.size(); ++i) from_cam(rig[i], &out[i]);
  });
}

int orc_split_rig(int64_t n_views, double test_fraction, uint64_t seed, int32_t* train,
                  int64_t* n_train, int32_t* test, int64_t* n_test) {
  return guarded([&] {
    RigSplit s = split_rig(static_cast<size_t>(n_views), test_fraction, seed);
    *n_train = static_cast<int64_t>(s.train.size());
    *n_test = static_cast<int64_t>(s.test.size());
    std::memcpy(train, s.train.data(), sizeof(int32_t) * s.train.size());
    std::memcpy(test, s.test.data(), sizeof(int32_t) * s.test.size());
  });
}

int orc_knn_mean(const double* points, int64_t n, int32_t k, double* out) {
  return guarded([&] {
    auto d = knn_mean_distances(to_cloud(points, nullptr, n), k);
    std::memcpy(out, d.data(), sizeof(double) * d.size());
  });
}

int orc_median_nn(const double* points, int64_t n, double* out) {
  return guarded([&] { *out = median_nn_spacing(to_cloud(points, nullptr, n)); });
}

int orc_seed_knn(const double* points, const double* colors, int64_t n, int32_t k,
                 double* params) {
  return guarded([&] {
    from_model(seed_gaussians(to_cloud(points, colors, n), ScaleRule::Knn, k), params);
  });
}

int orc_gt_model(const double* points, const double* colors, int64_t n, double scale,
                 double opacity, double* params) {
  return guarded([&] {
    from_model(ground_truth_model(to_cloud(points, colors, n), scale, opacity), params);
  });
}

int orc_rng_uniform(uint64_t seed, int64_t count, double* out) {
  return guarded([&] {
    Rng r(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = r.uniform();
  });
}

}  // extern "C"

// ---- float64 PLY (ply_io.hpp:89-221), reference only -----------------------
extern "C" int orc_write_splat_ply(const char* path, const double* params, int64_t n,
                                   int64_t iteration, int32_t origin) {
  return guarded([&] {
    SplatModel m = to_model(params, n);
    m.iteration = iteration;
    if (origin >= 0) m.origin_partition = origin;
    write_splat_ply(path, m);
  });
}

extern "C" int orc_read_splat_ply(const char* path, double* params, int64_t cap, int64_t* n,
                                  int64_t* iteration, int32_t* origin) {
  return guarded([&] {
    SplatModel m = read_splat_ply(path);
    *n = static_cast<int64_t>(m.size());
    *iteration = m.iteration;
    *origin = m.origin_partition ? *m.origin_partition : -1;
    if (params && cap >= *n) from_model(m, params);
  });
}

extern "C" int orc_write_cloud_ply(const char* path, const double* pos, const double* nrm,
                                   const double* col, int64_t n) {
  return guarded([&] {
    PointCloud pc;
    pc.points.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      SurfacePoint& p = pc.points[static_cast<size_t>(i)];
      p.position = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
      p.normal = {nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]};
      p.color = {col[3 * i], col[3 * i + 1], col[3 * i + 2]};
    }
    write_cloud_ply(path, pc);
  });
}
