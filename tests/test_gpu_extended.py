"""GPU parity beyond the single-view path: seeding, view synthesis, device
partitioning and merge, the tile-parallel render, and a config-1-scale
train step (99,726-point sphere isosurface, 256^2 views).
"""
import numpy as np
import pytest

from oracle import Oracle
from paper_2509_12138_b200 import api, scenes
from paper_2509_12138_b200.types import RenderConfig, SplatModel, TrainConfig, TrainView
from test_gpu_parity import assert_grads_close
from util import fp32_exact, random_cloud, random_scene
from util import test_camera as make_camera

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.fixture(scope="module")
def ctx():
    return api.Context(0)


def test_knn_and_median_bit_exact(orc, ctx):
    pts = random_cloud(3, 1500)
    for k in (1, 3, 5):
        np.testing.assert_array_equal(api.knn_mean_distances(pts, k, ctx=ctx),
                                      orc.knn_mean_distances(pts, k))
    assert api.median_nn_spacing(pts, ctx=ctx) == orc.median_nn_spacing(pts)
    surf, _, _ = scenes.sphere(4000)
    np.testing.assert_array_equal(api.knn_mean_distances(surf, 3, ctx=ctx),
                                  orc.knn_mean_distances(surf, 3))


def test_seed_and_gt_models(orc, ctx):
    pts, cols, _ = scenes.sphere(3000)
    a = api.seed_gaussians(pts, cols, 3, ctx=ctx).download().params
    b = orc.seed_gaussians(pts, cols).params.astype(np.float32).astype(np.float64)
    np.testing.assert_allclose(a, b, rtol=2e-7, atol=0)
    g = api.ground_truth_model(pts, cols, 0.01, 0.97, ctx=ctx).download().params
    h = orc.ground_truth_model(pts, cols, 0.01).params.astype(np.float32).astype(np.float64)
    np.testing.assert_allclose(g, h, rtol=2e-7, atol=0)


def test_view_synthesis_matches_make_train_view(orc, ctx):
    pts, cols, _ = scenes.sphere(6000)
    nn = orc.median_nn_spacing(pts)
    gt = orc.ground_truth_model(pts, cols, nn)
    gt = fp32_exact(gt)
    cams = scenes.rig_for_cloud(pts, 4, 2, 96)[:3]
    dgt = api.DeviceModel(ctx, gt)
    views = api.DeviceViews.synthesize(ctx, dgt, RenderConfig(), cams, pts, True, 2.0, 2.0)
    for i, cam in enumerate(cams):
        v = views.download(i)
        ref = orc.render(gt, cam, RenderConfig()).color
        assert np.max(np.abs(v.ground_truth - ref)) <= 1e-3
        np.testing.assert_array_equal(v.mask, orc.render_mask(pts, cam, 2.0, 2.0))


@pytest.mark.parametrize("nparts,margin", [(1, 0.25), (3, 0.15), (8, 0.3)])
def test_device_partition_bit_exact(orc, ctx, nparts, margin):
    pts = random_cloud(nparts + 9, 5000)
    pts[::13, 0] = pts[0, 0]
    pts[5, 0] = -0.0
    pts[6, 0] = 0.0
    a = api.partition_cloud(pts, nparts, margin, ctx=ctx)
    b = orc.partition_cloud(pts, nparts, margin)
    for pa, pb in zip(a, b):
        assert pa.cut_axis == pb.cut_axis and pa.cut_lo == pb.cut_lo and pa.cut_hi == pb.cut_hi
        np.testing.assert_array_equal(pa.owned_box, pb.owned_box)
        np.testing.assert_array_equal(pa.owned_indices, pb.owned_indices)
        np.testing.assert_array_equal(pa.ghost_indices, pb.ghost_indices)


def test_device_merge_matches_oracle(orc, ctx):
    pts = random_cloud(41, 400)
    parts = orc.partition_cloud(pts, 3, 0.2)
    rng = np.random.default_rng(1)
    models = [fp32_exact(SplatModel(rng.uniform(-1.2, 1.2, size=(50 + 7 * k, 14)), 4 + k, k))
              for k in range(3)]
    merged = api.merge_models(models, parts, ctx=ctx).download()
    keep = orc.merge_keep([m.params for m in models], parts)
    np.testing.assert_array_equal(merged.params, np.concatenate([m.params for m in models])[keep])
    assert merged.iteration == 6


def test_render_distributed_single_rank_equals_render(ctx):
    model = fp32_exact(random_scene(99, 300))
    model.params[:, 3:6] -= 1.5
    cam = make_camera(96)
    dm = api.DeviceModel(ctx, model)
    img, ms = api.render_distributed(None, dm, cam, RenderConfig())
    ref = api.render(dm, cam, RenderConfig(), ctx=ctx).color
    np.testing.assert_array_equal(img, ref)
    assert ms > 0


def test_config1_scale_train_step(orc, ctx):
    """Config 1 shape: 99,726-point sphere isosurface, GT at the median NN
    spacing, 256^2 views, kNN seeds; two train steps vs the oracle."""
    pts, cols, _ = scenes.sphere()
    nn = orc.median_nn_spacing(pts[:20000])  # O(N^2) oracle on a subset; value only sets scales
    gt = fp32_exact(orc.ground_truth_model(pts, cols, nn))
    cams = scenes.rig_for_cloud(pts, 16, 4, 256)[:2]
    seeds = fp32_exact(SplatModel(api.seed_gaussians(pts, cols, 3, ctx=ctx).download().params))
    views = [TrainView(c, orc.render(gt, c, RenderConfig()).color, orc.render_mask(pts, c, 2.0, 2.0))
             for c in cams]
    cfg = TrainConfig(iterations=2, seed=1)
    a = api.train_partition_full(seeds, views, cfg, ctx=ctx, loss_trace=True)
    b = orc.train_partition_full(seeds, views, cfg, loss_trace=True)
    # step 1 sees identical inputs; step 2 sees fp32 post-Adam params (<= 1e-4 relative)
    np.testing.assert_allclose(a.loss_trace[:1], b.loss_trace[:1], rtol=1e-6)
    np.testing.assert_allclose(a.loss_trace, b.loss_trace, rtol=1e-4)

    # One step: with epsilon = 1e-15 Adam moves every scalar by ~lr*sign(g)
    # (adam.hpp:84-91), so post-Adam parity holds wherever the reference
    # gradient is above the stated floor (1e-4 x the group's max |g|); below
    # it the sign is fp noise and a flip moves the scalar by 2*lr.
    cfg1 = TrainConfig(iterations=1, seed=1)
    a1 = api.train_partition_full(seeds, views, cfg1, ctx=ctx)
    b1 = orc.train_partition_full(seeds, views, cfg1)
    order = api.view_order(1, len(views), 1)
    v0 = views[int(order[0])]
    ref = orc.render(seeds, v0.cam, RenderConfig())
    g = orc.backward(seeds, v0.cam, RenderConfig(), ref,
                     orc.masked_loss(ref.color, v0, cfg1.loss_lambda).dL_dpixels).grads
    step_a, step_b = a1.model.params - seeds.params, b1.model.params - seeds.params
    flips = 0
    for name, sl in (("mu", slice(0, 3)), ("log_scale", slice(3, 6)), ("rot", slice(6, 10)),
                     ("opacity", slice(10, 11)), ("color", slice(11, 14))):
        gs = np.abs(g[:, sl])
        strong = gs >= 1e-4 * gs.max() if gs.max() > 0 else np.zeros_like(gs, bool)
        da, db = step_a[:, sl], step_b[:, sl]
        tol = 1e-4 * np.abs(db) + 1e-6 * np.abs(db).max()
        bad = np.abs(da - db) > tol
        assert not (bad & strong).any(), (name, int((bad & strong).sum()))
        flips += int(bad.sum())
    assert flips <= 0.005 * step_a.size, flips


@pytest.mark.parametrize("split_thr", [0.2, 0.0])
def test_train_with_densify_matches_oracle(orc, ctx, split_thr):
    """Clone / split / prune events on the device (trainer.hpp:47-107, 195-202):
    same model size and per-splat parameters as the oracle, which is pinned
    bit-exact to the reference (test_oracle_pin.test_train_densify_bit_exact)."""
    cam = make_camera(32)
    init = random_scene(45, 8)
    # a large anisotropic splat (an isotropic one has a pure-noise rotation
    # gradient, which Adam turns into +-lr steps in either implementation)
    init.params[0, 3:6] = np.log([0.5, 0.35, 0.25])
    init.params[1, 10] = -9.0
    init = fp32_exact(init)
    gt = orc.render(fp32_exact(random_scene(46, 8)), cam, RenderConfig()).color
    views = [TrainView(cam, gt, np.ones((32, 32)))]
    cfg = TrainConfig(iterations=60, seed=4, densify_interval=10, densify_grad_threshold=1e-5,
                      split_scale_threshold=split_thr)
    a = api.train_partition_full(init, views, cfg, ctx=ctx, loss_trace=True)
    b = orc.train_partition_full(init, views, cfg, loss_trace=True)
    assert len(a.model) == len(b.model) and len(a.model) != len(init)
    np.testing.assert_allclose(a.loss_trace, b.loss_trace, rtol=2e-3)
    np.testing.assert_allclose(a.model.params, b.model.params, rtol=0, atol=5e-3)


@pytest.mark.parametrize("scene", ["kingsnake", "random"])
def test_exact_submasks_change_nothing(ctx, scene):
    """The exact per-row sub-tile masks only skip (entry, sub-tile) hits that
    cannot composite: renders, contributor counts and gradients are
    bit-identical to the rect-only masks."""
    if scene == "kingsnake":
        pts, cols, _ = scenes.kingsnake(300_000, seed=3)
        model = api.seed_gaussians(pts, cols, 3, ctx=ctx).download()
        cams = scenes.rig_for_cloud(pts, 8, 4, 384)[::7]
    else:
        model = fp32_exact(random_scene(71, 3000))
        model.params[:, 3:6] += np.log(np.random.default_rng(5).uniform(0.05, 1.0, (3000, 3)))
        model = fp32_exact(model)
        cams = [make_camera(160)]
    rc = RenderConfig()
    outs = []
    for exact in (True, False):
        api.set_exact_masks(exact)
        try:
            res = []
            for cam in cams:
                r = api.render(model, cam, rc, ctx=ctx)
                dl = np.random.default_rng(9).normal(size=r.color.shape)
                g = api.backward(model, cam, rc, r, dl, ctx=ctx)
                res.append((r.color, r.per_pixel_contributor_count, g.grads, g.touch_count))
            outs.append(res)
        finally:
            api.set_exact_masks(True)
    for a, b in zip(*outs):
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("cluster", [40, 3000])
def test_near_coincident_depth_order(orc, ctx, cluster):
    """Many splats at (nearly) the same depth: exact ties, and depths closer
    than the 32-bit key quantum in shuffled index order. The order must still
    be the reference's (fp64 depth, index) order — short runs are fixed in
    place, long ones by a radix sort on the fp64 depth bits."""
    rng = np.random.default_rng(cluster)
    model = fp32_exact(random_scene(17, cluster + 500))
    c = model.params[:cluster].copy()
    c[:, 0:3] = [0.05, -0.03, 0.1]
    # every other splat nudged by one fp32 ulp in z: depth differences far
    # below the key quantum, in index order opposite to depth order
    nudge = rng.integers(0, 3, cluster).astype(np.float64)
    c[:, 2] = np.float32(0.1) + nudge * np.spacing(np.float32(0.1))
    model.params[:cluster] = c
    # one distant splat widens the depth range so the key quantum (range /
    # 2^32) exceeds the nudges: the whole cluster shares one key
    model.params[cluster, 0:3] = [0.0, 0.0, 40.0]
    model = fp32_exact(model)
    cam = make_camera(96)
    a = api.render(model, cam, RenderConfig(), ctx=ctx)
    b = orc.render(model, cam, RenderConfig())
    np.testing.assert_array_equal(a.splat_order, b.splat_order)
    assert np.max(np.abs(a.color - b.color)) <= 1e-3


@pytest.mark.parametrize("opacity", [-2.0, 1.5])
def test_long_tile_lists_split(orc, ctx, opacity):
    """A tile list of ~60k entries: the forward splits it into segments
    (segment products, incoming T, exact termination) and the backward walks
    them in parallel from checkpoints. Images, contributor counts and
    gradients follow the oracle; low opacity keeps most pixels alive through
    every segment, high opacity terminates them in the first one."""
    rng = np.random.default_rng(11)
    n = 60000
    p = np.zeros((n, 14))
    cam = make_camera(64)
    # tiny splats packed into a few tiles around the image centre
    p[:, 0] = rng.uniform(-0.02, 0.02, n)
    p[:, 1] = rng.uniform(-0.02, 0.02, n)
    p[:, 2] = rng.uniform(-0.3, 0.3, n)
    p[:, 3:6] = np.log(rng.uniform(0.001, 0.004, (n, 3)))
    q = rng.normal(size=(n, 4))
    p[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    p[:, 10] = opacity + rng.uniform(-0.5, 0.5, n)
    p[:, 11:14] = rng.uniform(0.1, 0.9, (n, 3))
    model = fp32_exact(SplatModel(p))
    counts, _ = api.bin_splats(model, cam, RenderConfig(), ctx=ctx, capacity=1 << 22)
    assert counts.max() > 40000  # the forward splits lists above 32768
    a = api.render(model, cam, RenderConfig(), ctx=ctx)
    b = orc.render(model, cam, RenderConfig())
    assert np.max(np.abs(a.color - b.color)) <= 1e-3
    nc_a, nc_b = np.asarray(a.per_pixel_contributor_count), np.asarray(b.per_pixel_contributor_count)
    np.testing.assert_array_equal(nc_a, nc_b)
    dl = np.random.default_rng(2).normal(size=a.color.shape) * 0.01
    ga = api.backward(model, cam, RenderConfig(), a, dl, ctx=ctx)
    gb = orc.backward(model, cam, RenderConfig(), b, dl)
    assert_grads_close(ga.grads, gb.grads)


@pytest.mark.parametrize("n", [1, 37, 600_001])
def test_model_transfer_round_trip(ctx, n):
    """Staged host<->device model copies (pinned chunks, worker pool, streaming
    stores): download(upload(P)) is P rounded to fp32, for ragged sizes that
    leave unaligned tails and span several 32 MiB chunks."""
    P = np.random.default_rng(n).normal(size=(n, 14)) * 10.0 ** np.random.default_rng(1).integers(-30, 30, size=(n, 14))
    dm = api.DeviceModel(ctx, SplatModel(P, 5, 2))
    out = dm.download()
    np.testing.assert_array_equal(out.params, P.astype(np.float32).astype(np.float64))
    assert out.iteration == 5 and out.origin_partition == 2
    dm.upload(SplatModel(P[: max(1, n // 2)]))
    np.testing.assert_array_equal(dm.download().params,
                                  P[: max(1, n // 2)].astype(np.float32).astype(np.float64))


def test_checkpoint_sink(orc, ctx):
    """CheckpointSink (trainer.hpp:119-120, 204-209): called every
    checkpoint_interval steps and once at the end with the model, its Adam
    state (serialize() = [step, size, m..., v...], adam.hpp:103-112), the
    model iteration and the step's loss."""
    cam = make_camera(40)
    target = fp32_exact(random_scene(24, 10))
    model = fp32_exact(random_scene(25, 10))
    model.origin_partition = 3
    view = TrainView(cam, orc.render(target, cam, RenderConfig()).color, np.ones((40, 40)))
    calls = []
    cfg = TrainConfig(iterations=12, seed=5, checkpoint_interval=5)
    res = api.train_partition_full(
        model, [view], cfg, ctx=ctx, loss_trace=True,
        checkpoint=lambda m, a, it, loss: calls.append((m, a.serialize(), it, loss)))
    assert [c[2] for c in calls] == [5, 10, 12]
    for m, payload, it, loss in calls:
        assert m.iteration == it and m.origin_partition == 3
        assert payload[0] == it and payload[1] == len(m) and len(payload) == 2 + 28 * len(m)
        assert loss == res.loss_trace[min(it, 12) - 1]
    np.testing.assert_array_equal(calls[-1][0].params, res.model.params)
    ref = orc.train_partition_full(model, [view], TrainConfig(iterations=12, seed=5))
    assert abs(ref.final_loss - res.final_loss) <= 1e-4 * ref.final_loss


@pytest.mark.parametrize("kind", ["rt", "rm"])
def test_device_heightfield_matches_numpy(ctx, kind):
    """The streamed device generator (dsg_heightfield_cloud) and its numpy
    restatement give the same cloud: transcendental results may differ by an
    ulp before the fp32 rounding, so a rare value moves by one fp32 ulp."""
    n = 300_001
    a = scenes.make_cloud(kind, n, seed=3, ctx=ctx)
    b = scenes.make_cloud(kind, n, seed=3)
    for x, y in zip(a, b):
        np.testing.assert_allclose(x, y, rtol=3e-7, atol=1e-9)
        assert np.mean(x != y) < 1e-3
    # any slice of the cloud depends only on (seed, index): a prefix of a
    # larger cloud with the same lattice side is identical
    np.testing.assert_array_equal(scenes.make_cloud(kind, n, seed=3, ctx=ctx)[0], a[0])


def _coincident_clusters(nclusters=1100, per=80):
    """nclusters clusters of `per` splats whose camera depths differ by less
    than the depth-key quantum, in reverse index order: every cluster is a
    long run of equal keys that needs the exact (fp64 depth, index) order."""
    rng = np.random.default_rng(5)
    P = np.zeros((nclusters * per, 14))
    side = int(np.ceil(np.sqrt(nclusters)))
    k = 0
    for c in range(nclusters):
        cx = ((c % side) / side - 0.5) * 1.6
        cy = ((c // side) / side - 0.5) * 1.6
        cz = rng.uniform(0.0, 8.0)
        for j in range(per):
            P[k, 0:3] = [cx - j * 2.0 ** -16, cy, cz]
            k += 1
    P[:, 3:6] = np.log(0.002)
    P[:, 6] = 1.0
    P[:, 10] = 2.0
    P[:, 11:14] = 0.5
    return fp32_exact(SplatModel(P))


def test_more_long_runs_than_the_per_run_path(orc, ctx):
    """More than kLongCap (1024) long near-coincident runs: the whole visible
    set is sorted by (fp64 depth bits, index) instead of failing (round 1
    raised InvalidArgument here). 1053 such runs in this scene (checked on
    the CPU by replaying the device's key quantisation)."""
    from paper_2509_12138_b200.types import Camera
    m = _coincident_clusters()
    cam = Camera((0.0, 0.0, -3.0), (3e-7, 0.0, 0.0), (0.0, 1.0, 0.0), 1.2, 128, 128, 0.1, 50.0)
    a = api.render(m, cam, RenderConfig(), ctx=ctx)
    b = orc.render(m, cam, RenderConfig())
    np.testing.assert_array_equal(a.splat_order, b.splat_order)
    assert np.max(np.abs(a.color - b.color)) <= 1e-3
    np.testing.assert_array_equal(a.per_pixel_contributor_count, b.per_pixel_contributor_count)


def test_view_sources_train_identically(orc, ctx):
    """The three view sources of dsg_train — device-resident views, planar
    views streamed from pinned host memory (dsg_views_create_host, used by
    the partitioned bench) and reference-layout TrainViews converted per
    step (dsg_views_create_host_ref, used by train_partition_full) — give
    bit-identical trajectories."""
    pts, cols, _ = scenes.sphere(6000)
    cams = scenes.rig_for_cloud(pts, 4, 2, 96)[:5]
    gt = api.DeviceModel(ctx, fp32_exact(orc.ground_truth_model(pts, cols, 0.01)))
    dviews = api.DeviceViews.synthesize(ctx, gt, RenderConfig(), cams, pts, True, 2.0, 2.0)
    seeds = api.seed_gaussians(pts, cols, 3, ctx=ctx).download()
    cfg = TrainConfig(iterations=9, seed=4, densify_interval=0)
    runs = []
    dm = api.DeviceModel(ctx, seeds)
    runs.append(api.train_device(dm, dviews, cfg, loss_trace=True)[1])
    p0 = dm.download().params
    planar = [dviews.download_planar(i, pin=True) for i in range(len(cams))]
    hv = api.HostViews(ctx, dviews.cams, [g for g, _ in planar], [m for _, m in planar])
    dm.upload(seeds)
    runs.append(api.train_device(dm, hv, cfg, loss_trace=True)[1])
    p1 = dm.download().params
    tv = [dviews.download(i) for i in range(len(cams))]
    r = api.train_partition_full(seeds, tv, cfg, ctx=ctx, loss_trace=True)
    runs.append(r.loss_trace)
    np.testing.assert_array_equal(runs[0], runs[1])
    np.testing.assert_array_equal(runs[0], runs[2])
    np.testing.assert_array_equal(p0, p1)
    np.testing.assert_array_equal(p0, r.model.params)


def test_frame_work_counts_composited_pairs(ctx):
    """dsg_frame_work: C = sum of n_contrib of the last forward (the blend
    kernels' work count in the bench's roofline), plus the fix-up counters."""
    m = fp32_exact(random_scene(99, 300))
    m.params[:, 3:6] -= 1.5
    r = api.render(m, make_camera(64), RenderConfig(), ctx=ctx)
    w = api.frame_work(ctx)
    assert w["composited"] == int(np.sum(r.per_pixel_contributor_count)) > 0
    assert 0 <= w["term_changed"] <= w["term_fixups"]


FUSE_SCRIPT = r"""
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
from paper_2509_12138_b200 import api, scenes
from paper_2509_12138_b200.types import RenderConfig, TrainConfig
ctx = api.Context(0)
pts, cols, _ = scenes.kingsnake(30000, seed=2)
nn = api.median_nn_spacing(pts, ctx=ctx)
rig = scenes.rig_for_cloud(pts, 8, 4, 128)
gt = api.ground_truth_model(pts, cols, nn, 0.97, ctx=ctx)
views = api.DeviceViews.synthesize(ctx, gt, RenderConfig(), rig[:6], pts, True, 2.0, 2.0)
dm = api.seed_gaussians(pts, cols, 3, ctx=ctx)
cfg = TrainConfig(iterations=16, seed=3, densify_interval=4, densify_grad_threshold=1e-5)
fl, trace = api.train_device(dm, views, cfg, loss_trace=True)
m, v, st = dm.adam_state()
np.savez(sys.argv[1], params=dm.download().params, m=m, v=v, trace=trace, step=np.array([st]))
"""


def test_fused_chain_adam_bit_identical(tmp_path):
    """dsg_train's fused chain + Adam kernel (gradients never stored) against
    the separate k_chain and k_adam launches (DSG_FUSE_ADAM=0): parameters,
    moments and loss trace bit-identical over 16 steps with densification."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "fuse.py"
    script.write_text(FUSE_SCRIPT)
    out = {}
    for flag in ("0", "1"):
        path = str(tmp_path / f"fuse{flag}.npz")
        env = dict(os.environ, ROOT=root, DSG_FUSE_ADAM=flag)
        r = subprocess.run([sys.executable, str(script), path], capture_output=True, text=True,
                           timeout=300, env=env)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        out[flag] = np.load(path)
    a, b = out["0"], out["1"]
    assert a["params"].shape == b["params"].shape
    for k in ("params", "m", "v", "trace", "step"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
