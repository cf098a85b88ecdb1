"""Parity at the benched and named configurations (BASELINE configs 1-5).

Every check in tests/scale_parity.py (splat order and per-tile lists
bit-exact, image <= 1e-3, gradients <= 1e-4 relative with the per-group
floor, touch counts exact, Adam, one full train iteration) runs on:

  * config 1: the 99,726-point sphere isosurface, 256^2 view, kNN seeds
  * config 2: the 4M-Gaussian Kingsnake partition, 1024^2 view — the
    workload bench.py times
  * config 3: one 8-way RT partition (18.2M-point cloud, auto ghosts):
    owned / ghost lists and cuts bit-exact against partition_cloud
    (partition.hpp:42-104), the partition's background mask bit-exact
    (render.hpp:210-233), and the step checks on its seeds
  * config 4: the 106.7M RM cloud in 8 slabs (every partition bit-exact)
    and one 13.4M-splat partition's step at 2048^2
  * config 5: the RT partitions' merge and the merged model's 4K render

Inputs are built the way bench.py builds them (device kNN seeds and
median NN spacing, device-synthesized GT views); the device values are
fp32, and the checker receives exactly those values. The checker is
oracle/_ref (the reference compiled unchanged) when present.
"""
import json
import os

import numpy as np
import pytest

from paper_2509_12138_b200 import api, scenes
from paper_2509_12138_b200.types import RenderConfig, SplatModel, TrainConfig
from scale_parity import checker, step_parity

pytestmark = pytest.mark.gpu

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


@pytest.fixture(scope="module")
def ctx():
    return api.Context(0)


@pytest.fixture(scope="module")
def ref():
    return checker()[0]


def _record(name, rep):
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"scale_parity_{name}.json"), "w") as f:
        json.dump(rep, f, indent=1)


def _inputs(ctx, pts, cols, az, el, res):
    """bench.py's per-partition setup: median NN, GT model, seeds, first
    scheduled view (trainer.hpp:157-163) synthesized on the device."""
    nn = api.median_nn_spacing(pts, ctx=ctx)
    rig = scenes.rig_for_cloud(pts, az, el, res)
    from bench import split_rig
    train_idx, _ = split_rig(len(rig), 0.1, 1)
    cams = [rig[i] for i in train_idx]
    v0 = int(api.view_order(1, len(cams), 1)[0])
    gt = api.ground_truth_model(pts, cols, nn, 0.97, ctx=ctx)
    views = api.DeviceViews.synthesize(ctx, gt, RenderConfig(), [cams[v0]], pts, True, 2.0, 2.0)
    view = views.download(0)
    seeds = api.seed_gaussians(pts, cols, 3, ctx=ctx).download()
    return SplatModel(np.ascontiguousarray(seeds.params)), view, nn


def _assert_pass(rep):
    assert rep["splat_order_bit_exact"], rep
    assert rep["tile_counts_bit_exact"] and rep["tile_lists_bit_exact"], rep
    assert rep["img_max_abs"] <= 1e-3 and rep["alpha_max_abs"] <= 1e-3, rep
    assert rep["grad_worst_over_tol"] <= 1.0, rep["grads"]
    assert rep["touch_count_exact"], rep
    assert rep["adam_worst_over_tol"] <= 1.0, rep
    assert rep["train_step_bad_above_floor"] == 0, rep
    # the loss-conditioned exclusion stays a small fraction of the step, and
    # the two dL images agree away from the L1 kinks
    assert rep["train_step_loss_conditioned_excluded"] <= 1e-3 * rep["train_step_scalars"], rep
    # (the SSIM gradient amplifies the ~1e-6 image difference by ~1/C2)
    assert rep["dL_max_rel_off_kinks"] <= 1e-3, rep
    assert rep["loss_rel"] <= 1e-4, rep
    # contributor counts: exact (termination near the floor is re-decided in fp64)
    assert rep["ncontrib_mismatch_px"] == 0, rep
    assert rep["pass"]


def test_config1_sphere_step_parity(ctx, ref):
    pts, cols, _ = scenes.sphere()
    model, view, _ = _inputs(ctx, pts, cols, 16, 4, 256)
    rep = step_parity(ctx, ref, model, view, TrainConfig(iterations=1, seed=1))
    _record("config1", rep)
    _assert_pass(rep)


def test_config2_kingsnake_step_parity(ctx, ref):
    pts, cols, _ = scenes.kingsnake(scenes.SIZES["kingsnake"], seed=1, turns=6.0)
    model, view, _ = _inputs(ctx, pts, cols, 28, 16, 1024)
    assert len(model) == 4_000_000
    rep = step_parity(ctx, ref, model, view, TrainConfig(iterations=1, seed=1))
    _record("config2", rep)
    _assert_pass(rep)


def test_config2_knn_seeds_at_scale(ctx):
    """knn_mean_distances (seed.hpp:16-35) on the 4M cloud: the device grid
    kNN against an independent exact kNN (scipy cKDTree), summing the k
    smallest fp64 distances in ascending order as the reference does."""
    from scipy.spatial import cKDTree
    pts, _, _ = scenes.kingsnake(scenes.SIZES["kingsnake"], seed=1, turns=6.0)
    dev = api.knn_mean_distances(pts, 3, ctx=ctx)
    d, _ = cKDTree(pts).query(pts, k=4, workers=os.cpu_count() or 1)
    host = (d[:, 1] + d[:, 2] + d[:, 3]) / 3.0
    np.testing.assert_array_equal(dev, host)
    nn1 = np.sort(d[:, 1])[len(pts) // 2]
    assert api.median_nn_spacing(pts, ctx=ctx) == nn1


@pytest.fixture(scope="module")
def rt_cloud(ctx):
    return scenes.make_cloud("rt", scenes.SIZES["rt"], seed=1, ctx=ctx)  # device generator


def test_config3_rt_partition_bit_exact(ctx, ref, rt_cloud):
    pts, cols, _ = rt_cloud
    nn = api.median_nn_spacing(pts, ctx=ctx)
    margin = 3.0 * nn
    a = api.partition_cloud(pts, 8, margin, ctx=ctx)
    b = ref.partition_cloud(pts, 8, margin)
    summary = []
    for pa, pb in zip(a, b):
        assert pa.cut_axis == pb.cut_axis
        assert pa.cut_lo == pb.cut_lo and pa.cut_hi == pb.cut_hi
        np.testing.assert_array_equal(pa.owned_indices, pb.owned_indices)
        np.testing.assert_array_equal(pa.ghost_indices, pb.ghost_indices)
        np.testing.assert_array_equal(pa.owned_box, pb.owned_box)
        summary.append([int(len(pb.owned_indices)), int(len(pb.ghost_indices))])
    _record("config3_partition", {"points": int(len(pts)), "margin": margin,
                                  "owned_ghost": summary, "bit_exact": True})


def test_config3_rt_partition_mask_and_step(ctx, ref, rt_cloud):
    pts, cols, _ = rt_cloud
    nn = api.median_nn_spacing(pts, ctx=ctx)
    parts = api.partition_cloud(pts, 8, 3.0 * nn, ctx=ctx)
    part = parts[3]
    idx = np.concatenate([part.owned_indices, part.ghost_indices]).astype(np.int64)
    ppts, pcols = np.ascontiguousarray(pts[idx]), np.ascontiguousarray(cols[idx])
    rig = scenes.rig_for_cloud(pts, 28, 16, 1024)  # global rig (runtime.hpp:137)
    cam = rig[37]
    np.testing.assert_array_equal(api.render_mask(ppts, cam, 2.0, 2.0, ctx=ctx),
                                  ref.render_mask(ppts, cam, 2.0, 2.0))
    gt = api.ground_truth_model(ppts, pcols, nn, 0.97, ctx=ctx)
    views = api.DeviceViews.synthesize(ctx, gt, RenderConfig(), [cam], ppts, True, 2.0, 2.0)
    view = views.download(0)
    seeds = api.seed_gaussians(ppts, pcols, 3, ctx=ctx).download()
    model = SplatModel(np.ascontiguousarray(seeds.params))
    rep = step_parity(ctx, ref, model, view, TrainConfig(iterations=1, seed=4))
    rep["partition"] = 3
    rep["owned"], rep["ghosts"] = int(len(part.owned_indices)), int(len(part.ghost_indices))
    _record("config3_step", rep)
    _assert_pass(rep)


def test_config2_three_step_trajectory(ctx, ref):
    """Three training iterations of the benched 4M partition (trainer.hpp:
    173-207: seeded view order, lr_mu decay, Adam) on three of its 1024^2
    views, on both sides: the loss trace agrees to 1e-4 relative. Step 1
    sees identical inputs; later steps see the fp32 post-Adam parameters,
    whose only visible differences are the noise-level gradient components
    where Adam's epsilon = 1e-15 moves a scalar by +-lr either way."""
    import os as _os
    pts, cols, _ = scenes.kingsnake(scenes.SIZES["kingsnake"], seed=1, turns=6.0)
    nn = api.median_nn_spacing(pts, ctx=ctx)
    rig = scenes.rig_for_cloud(pts, 28, 16, 1024)
    from bench import split_rig
    train_idx, _ = split_rig(len(rig), 0.1, 1)
    cams = [rig[i] for i in train_idx[:3]]
    gt = api.ground_truth_model(pts, cols, nn, 0.97, ctx=ctx)
    views = api.DeviceViews.synthesize(ctx, gt, RenderConfig(), cams, pts, True, 2.0, 2.0)
    tv = [views.download(k) for k in range(3)]
    seeds = SplatModel(np.ascontiguousarray(api.seed_gaussians(pts, cols, 3, ctx=ctx).download().params))
    cfg = TrainConfig(iterations=3, seed=1)
    a = api.train_partition_full(seeds, tv, cfg, ctx=ctx, loss_trace=True)
    b = ref.train_partition_full(seeds, tv, cfg, shards=_os.cpu_count() or 1, loss_trace=True)
    _record("config2_trajectory", {"device": a.loss_trace.tolist(), "reference": b.loss_trace.tolist()})
    np.testing.assert_allclose(a.loss_trace, b.loss_trace, rtol=1e-4)


def test_config5_merged_4k_render(ctx, ref, rt_cloud):
    """Config 5's path at RT scale: the 8 partitions' seed models ghost-trimmed
    and merged on the device (merge_models, partition.hpp:109-126), then the
    merged 18M-splat model rendered at 3840x2160 (explicit camera, as
    runtime.hpp:476-520 renders the merged model). Against the reference:
    merge bit-exact (fp32-exact inputs), splat order bit-exact, image <= 1e-3,
    contributor counts exact. (The 106.7M RM model is beyond what the CPU
    reference renders in a test's time.)"""
    from paper_2509_12138_b200.types import Camera
    from host_partition import merge_models
    pts, cols, _ = rt_cloud
    nn = api.median_nn_spacing(pts, ctx=ctx)
    parts = api.partition_cloud(pts, 8, 3.0 * nn, ctx=ctx)
    models, hosts = [], []
    for k, p in enumerate(parts):
        idx = np.concatenate([p.owned_indices, p.ghost_indices]).astype(np.int64)
        dm = api.seed_gaussians(np.ascontiguousarray(pts[idx]), np.ascontiguousarray(cols[idx]), 3,
                                ctx=ctx)
        h = dm.download()
        h.origin_partition = k
        models.append(dm)
        hosts.append(h)
    merged = api.merge_models(models, parts, ctx=ctx).download()
    expect = merge_models(hosts, parts)
    np.testing.assert_array_equal(merged.params, expect.params)
    del models
    c = (pts.min(0) + pts.max(0)) * 0.5
    rig = scenes.rig_for_cloud(pts, 28, 16, 1024)
    cam = Camera(rig[0].position, tuple(float(v) for v in c), (0.0, 1.0, 0.0), 0.9, 3840, 2160,
                 rig[0].near, rig[0].far)
    a = api.render(merged, cam, RenderConfig(), ctx=ctx)
    b = ref.render(merged, cam, RenderConfig())
    rep = {"merged": int(len(merged)), "splat_order_bit_exact": bool(np.array_equal(a.splat_order, b.splat_order)),
           "img_max_abs": float(np.max(np.abs(a.color - b.color))),
           "ncontrib_mismatch_px": int(np.sum(a.per_pixel_contributor_count != b.per_pixel_contributor_count))}
    _record("config5_rt_merged_4k", rep)
    assert rep["splat_order_bit_exact"], rep
    assert rep["img_max_abs"] <= 1e-3, rep
    assert rep["ncontrib_mismatch_px"] == 0, rep


def test_config4_rm_partition_and_step(ctx, ref):
    """Config 4's shape: the 106.7M-point RM cloud (device generator) in 8
    slabs — owned / ghost lists and cuts of every partition bit-exact against
    partition_cloud — then one partition's mask, GT view and seeds at 2048^2
    and the full step check (lists, order, image, n_contrib, gradients, Adam,
    one train iteration) against the reference on its 13.4M splats."""
    pts, cols, _ = scenes.make_cloud("rm", scenes.SIZES["rm"], seed=1, ctx=ctx)
    nn = api.median_nn_spacing(pts, ctx=ctx)
    margin = 3.0 * nn
    a = api.partition_cloud(pts, 8, margin, ctx=ctx)
    b = ref.partition_cloud(pts, 8, margin)
    summary = []
    for pa, pb in zip(a, b):
        assert pa.cut_axis == pb.cut_axis
        assert pa.cut_lo == pb.cut_lo and pa.cut_hi == pb.cut_hi
        np.testing.assert_array_equal(pa.owned_indices, pb.owned_indices)
        np.testing.assert_array_equal(pa.ghost_indices, pb.ghost_indices)
        summary.append([int(len(pb.owned_indices)), int(len(pb.ghost_indices))])
    del b
    part = a[5]
    idx = np.concatenate([part.owned_indices, part.ghost_indices]).astype(np.int64)
    ppts, pcols = np.ascontiguousarray(pts[idx]), np.ascontiguousarray(cols[idx])
    rig = scenes.rig_for_cloud(pts, 28, 16, 2048)  # global rig (runtime.hpp:137)
    del pts, cols, a
    cam = rig[37]
    np.testing.assert_array_equal(api.render_mask(ppts, cam, 2.0, 2.0, ctx=ctx),
                                  ref.render_mask(ppts, cam, 2.0, 2.0))
    gt = api.ground_truth_model(ppts, pcols, nn, 0.97, ctx=ctx)
    views = api.DeviceViews.synthesize(ctx, gt, RenderConfig(), [cam], ppts, True, 2.0, 2.0)
    view = views.download(0)
    del views, gt
    seeds = api.seed_gaussians(ppts, pcols, 3, ctx=ctx).download()
    model = SplatModel(np.ascontiguousarray(seeds.params))
    rep = step_parity(ctx, ref, model, view, TrainConfig(iterations=1, seed=6))
    rep["partition"] = 5
    rep["owned"], rep["ghosts"] = int(len(part.owned_indices)), int(len(part.ghost_indices))
    rep["partitions_owned_ghost"] = summary
    _record("config4_rm", rep)
    _assert_pass(rep)
