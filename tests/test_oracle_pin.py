"""Pin the oracle restatement to the reference itself (CPU, no GPU).

oracle/liboracle.so (this repo's restatement) against oracle/_ref (the
unmodified reference headers compiled here): every output of the path must be
BIT-identical on the same inputs — the restatement keeps the reference's
floating-point evaluation order (oracle/oracle.cpp header).
"""
import numpy as np
import pytest

from oracle import Oracle, Reference, has_reference
from paper_2509_12138_b200.types import Camera, RenderConfig, SplatModel, TrainConfig, TrainView
from util import Rng, disc_mask, fd_scene, full_mask, offset_ground_truth, random_cloud, random_scene
from util import smooth_config
from util import test_camera as make_camera

pytestmark = pytest.mark.skipif(not has_reference(), reason="oracle/_ref not built (no /root/reference)")


@pytest.fixture(scope="module")
def impls():
    return Oracle(), Reference()


def _eq(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape
    assert np.array_equal(a, b), f"max diff {np.max(np.abs(a.astype(float) - b.astype(float)))}"


def _scenes():
    cam = make_camera(48)
    out = []
    for seed in (21, 22, 23, 31, 55):
        out.append((random_scene(seed, 12), cam, RenderConfig()))
    out.append((fd_scene(7, 3), make_camera(32), smooth_config()))
    big = random_scene(99, 200)
    big.params[:, 3:6] -= 1.5  # small splats: many tiles, many culls near edges
    out.append((big, make_camera(64), RenderConfig(background=(0.2, 0.3, 0.4))))
    return out


@pytest.mark.parametrize("k", range(7))
def test_render_bit_exact(impls, k):
    o, r = impls
    model, cam, cfg = _scenes()[k]
    a = o.render(model, cam, cfg)
    b = r.render(model, cam, cfg)
    _eq(a.color, b.color)
    _eq(a.alpha, b.alpha)
    _eq(a.per_pixel_contributor_count, b.per_pixel_contributor_count)
    _eq(a.splat_order, b.splat_order)
    pa, pb = o.prepare(model, cam, cfg), r.prepare(model, cam, cfg)
    for key in pa:
        _eq(pa[key], pb[key])
    ca, ea = o.bin(model, cam, cfg)
    cb, eb = r.bin(model, cam, cfg)
    _eq(ca, cb)
    _eq(ea, eb)


@pytest.mark.parametrize("lam", [0.0, 0.2, 1.0])
def test_loss_bit_exact(impls, lam):
    o, r = impls
    rng = np.random.default_rng(3)
    a = rng.random((24, 20, 3))
    b = rng.random((24, 20, 3))
    view = TrainView(Camera(width=20, height=24), b, disc_mask(20, 24, 9.0, 12.0, 8.0))
    la, lb = o.masked_loss(a, view, lam), r.masked_loss(a, view, lam)
    assert la.loss == lb.loss
    _eq(la.dL_dpixels, lb.dL_dpixels)


@pytest.mark.parametrize("k", range(7))
def test_backward_bit_exact(impls, k):
    o, r = impls
    model, cam, cfg = _scenes()[k]
    out = r.render(model, cam, cfg)
    gt = offset_ground_truth(r.render, model, cam, cfg, 7 + k)
    view = TrainView(cam, gt, disc_mask(cam.width, cam.height, 20.0, 22.0, 15.0))
    lr = r.masked_loss(out.color, view, 0.2)
    ga = o.backward(model, cam, cfg, out, lr.dL_dpixels)
    gb = r.backward(model, cam, cfg, out, lr.dL_dpixels)
    _eq(ga.grads, gb.grads)
    _eq(ga.d_mean2d, gb.d_mean2d)
    _eq(ga.touch_count, gb.touch_count)


def test_adam_bit_exact(impls):
    o, r = impls
    rng = np.random.default_rng(5)
    P = random_scene(3, 50).params
    G = rng.normal(size=P.shape) * 1e-3
    G[::7] = 0.0
    res = []
    for impl in (o, r):
        p = P.copy()
        m = np.zeros_like(P)
        v = np.zeros_like(P)
        st = impl.adam_step(p, G, m, v, 0, (1e-3, 5e-3, 1e-3, 5e-2, 5e-3))
        res.append((p, m, v, st))
    for x, y in zip(res[0], res[1]):
        _eq(x, y)


def test_train_bit_exact(impls):
    o, r = impls
    cam = make_camera(32)
    init = random_scene(23, 6)
    gt = r.render(random_scene(24, 6), cam, RenderConfig()).color
    view = TrainView(cam, gt, full_mask(32, 32))
    cfg = TrainConfig(iterations=25, seed=9)
    a = o.train_partition_full(init, [view], cfg, loss_trace=True)
    b = r.train_partition_full(init, [view], cfg, loss_trace=True)
    _eq(a.model.params, b.model.params)
    assert a.final_loss == b.final_loss
    _eq(a.loss_trace, b.loss_trace)


def test_train_densify_bit_exact(impls):
    # densify fires at it+1 = 10, 20 (< 0.5 * 60): clone/split/prune paths.
    o, r = impls
    cam = make_camera(32)
    init = random_scene(45, 8)
    init.params[0, 3:6] = np.log(0.5)
    init.params[1, 10] = -9.0
    gt = r.render(random_scene(46, 8), cam, RenderConfig()).color
    views = [TrainView(cam, gt, full_mask(32, 32))]
    cfg = TrainConfig(iterations=60, seed=4, densify_interval=10, densify_grad_threshold=1e-5,
                      split_scale_threshold=0.2)
    a = o.train_partition_full(init, views, cfg)
    b = r.train_partition_full(init, views, cfg)
    assert len(a.model) == len(b.model) and len(a.model) != len(init)
    _eq(a.model.params, b.model.params)


def test_mask_bit_exact(impls):
    o, r = impls
    cam = make_camera(48)
    pts = random_cloud(9, 300, (-1.2, -1.2, -1.2), (1.2, 1.2, 1.2))
    for fp, dil in ((2.0, 2.0), (0.5, 0.0), (3.3, 1.7)):
        _eq(o.render_mask(pts, cam, fp, dil), r.render_mask(pts, cam, fp, dil))


@pytest.mark.parametrize("nparts,margin", [(1, 0.25), (2, 0.0), (3, 0.15), (4, 0.2), (8, 0.3)])
def test_partition_bit_exact(impls, nparts, margin):
    o, r = impls
    pts = random_cloud(nparts + 5, 337)
    pts[::11, 0] = pts[0, 0]  # ties on the cut axis
    a = o.partition_cloud(pts, nparts, margin)
    b = r.partition_cloud(pts, nparts, margin)
    for pa, pb in zip(a, b):
        assert pa.cut_axis == pb.cut_axis and pa.cut_lo == pb.cut_lo and pa.cut_hi == pb.cut_hi
        _eq(pa.owned_box, pb.owned_box)
        _eq(pa.owned_indices, pb.owned_indices)
        _eq(pa.ghost_indices, pb.ghost_indices)


def test_merge_bit_exact(impls):
    o, r = impls
    pts = random_cloud(41, 200)
    parts = r.partition_cloud(pts, 3, 0.2)
    rng = np.random.default_rng(1)
    models = [rng.uniform(-1.2, 1.2, size=(40 + 3 * k, 14)) for k in range(3)]
    _eq(o.merge_keep(models, parts), r.merge_keep(models, parts))


def test_rig_and_split_bit_exact(impls):
    o, r = impls
    for args in (((0.5, -1.0, 2.0), 3.25, 7, 5, 32), ((0, 0, 0), 2.5, 28, 16, 64),
                 ((1, 2, 3), 2.0, 1, 1, 64)):
        ca = o.build_orbital_cameras(*args)
        cb = r.build_orbital_cameras(*args)
        assert ca == cb
    for n, frac, seed in ((64, 0.1, 1), (28, 4 / 28, 11), (448, 0.1, 3), (1, 0.5, 2)):
        ta, sa = o.split_rig(n, frac, seed)
        tb, sb = r.split_rig(n, frac, seed)
        _eq(ta, tb)
        _eq(sa, sb)


def test_seed_and_gt_bit_exact(impls):
    o, r = impls
    pts = random_cloud(3, 400)
    cols = random_cloud(4, 400, (0, 0, 0), (1, 1, 1))
    _eq(o.knn_mean_distances(pts, 3), r.knn_mean_distances(pts, 3))
    assert o.median_nn_spacing(pts) == r.median_nn_spacing(pts)
    _eq(o.seed_gaussians(pts, cols).params, r.seed_gaussians(pts, cols).params)
    _eq(o.ground_truth_model(pts, cols, 0.0123).params, r.ground_truth_model(pts, cols, 0.0123).params)


def test_rng_stream_matches(impls):
    o, r = impls
    _eq(o.rng_uniform(77, 100), r.rng_uniform(77, 100))
    py = Rng(77)
    _eq(o.rng_uniform(77, 100), np.array([py.uniform() for _ in range(100)]))


def test_errors_match(impls):
    o, r = impls
    from paper_2509_12138_b200.types import DsplatError
    cam = make_camera(32)
    model = random_scene(5, 2)
    out = r.render(model, cam, RenderConfig())
    model.iteration = 1
    for impl in (o, r):
        with pytest.raises(DsplatError, match="StaleForward"):
            impl.backward(model, cam, RenderConfig(), out, np.zeros((32, 32, 3)))
        with pytest.raises(DsplatError, match="EmptyCloud"):
            impl.partition_cloud(np.zeros((0, 3)), 2, 0.1)
        with pytest.raises(DsplatError, match="InvalidArgument"):
            impl.render_mask(np.zeros((1, 3)), cam, 0.2, 0.0)
        with pytest.raises(DsplatError, match="NoViews"):
            impl.train_partition_full(model, [], TrainConfig())
        with pytest.raises(DsplatError, match="InvalidRig"):
            impl.build_orbital_cameras((0, 0, 0), 0.0, 4, 4, 64)
