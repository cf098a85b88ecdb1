"""GPU parity: the CUDA path (through the libdsg C ABI) against the CPU oracle.

Tolerances are the north star's (BASELINE.json):
  * tile-overlap counts, sorted per-tile key lists, splat order, masks: bit-exact
  * rendered images: max abs <= 1e-3 per channel
  * gradients / post-Adam parameters: <= 1e-4 relative, with an absolute floor
    per parameter group of GRAD_FLOOR x (max |reference| in that group) —
    fp32 device arithmetic against an fp64 oracle cannot resolve components
    that are pure cancellation noise (SURVEY §7 hard part 3).
Inputs are fp32-exact (util.fp32_exact) so both sides see identical values.
"""
import numpy as np
import pytest

from oracle import Oracle
from paper_2509_12138_b200 import api
from paper_2509_12138_b200.types import (DsplatError, GroupRates, RenderConfig, SplatModel,
                                         TrainConfig, TrainView)
from util import (disc_mask, fd_scene, fp32_exact, full_mask, offset_ground_truth, random_cloud,
                  random_scene, smooth_config)
from util import test_camera as make_camera

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-3
GRAD_RTOL = 1e-4
GRAD_FLOOR = 1e-5
GROUPS = {"mu": slice(0, 3), "log_scale": slice(3, 6), "rot": slice(6, 10), "opacity": slice(10, 11),
          "color": slice(11, 14)}


def assert_grads_close(g_dev, g_ref, rtol=GRAD_RTOL, floor=GRAD_FLOOR):
    for name, sl in GROUPS.items():
        a, b = g_dev[:, sl], g_ref[:, sl]
        scale = np.max(np.abs(b)) if b.size else 0.0
        tol = rtol * np.maximum(np.abs(a), np.abs(b)) + floor * scale
        bad = np.abs(a - b) > tol
        assert not bad.any(), (f"{name}: {bad.sum()} of {bad.size} out of tolerance; worst "
                               f"{np.max(np.abs(a - b) - tol):.3g} (scale {scale:.3g})")


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.fixture(scope="module")
def ctx():
    return api.Context(0)


def sphere_model(n=4000, seed=3, scale=0.01, opacity_logit=0.0):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    P = np.zeros((n, 14))
    P[:, 0:3] = 0.35 * v
    P[:, 3:6] = np.log(scale)
    P[:, 6] = 1.0
    P[:, 10] = opacity_logit
    P[:, 11:14] = 0.35 + 0.3 * (0.5 + 0.5 * v)
    return fp32_exact(SplatModel(P))


def scenes():
    out = []
    for seed in (21, 22, 23, 31, 55):
        out.append((fp32_exact(random_scene(seed, 12)), make_camera(48), RenderConfig()))
    out.append((fp32_exact(fd_scene(7, 3)), make_camera(32), smooth_config()))
    big = random_scene(99, 300)
    big.params[:, 3:6] -= 1.5
    out.append((fp32_exact(big), make_camera(64), RenderConfig(background=(0.2, 0.3, 0.4))))
    cam = make_camera(128)
    cam.position = (0.3, 0.4, -1.6)
    out.append((sphere_model(), cam, RenderConfig()))
    out.append((sphere_model(6000, 4, 0.004, 3.5), make_camera(256), RenderConfig()))
    return out


SCENES = scenes()


@pytest.mark.parametrize("k", range(len(SCENES)))
def test_render_parity(orc, ctx, k):
    model, cam, cfg = SCENES[k]
    a = api.render(model, cam, cfg, ctx=ctx)
    b = orc.render(model, cam, cfg)
    np.testing.assert_array_equal(a.splat_order, b.splat_order)
    assert np.max(np.abs(a.color - b.color)) <= IMG_TOL
    assert np.max(np.abs(a.alpha - b.alpha)) <= IMG_TOL
    # contributor counts: exact (pixels whose fp32 T lands near the floor are
    # re-walked in fp64 by k_term_fixup)
    np.testing.assert_array_equal(a.per_pixel_contributor_count, b.per_pixel_contributor_count)


@pytest.mark.parametrize("k", range(len(SCENES)))
def test_tile_lists_bit_exact(orc, ctx, k):
    model, cam, cfg = SCENES[k]
    cfg16 = RenderConfig(**{**cfg.__dict__, "tile_size": 16})
    ca, ea = api.bin_splats(model, cam, cfg16, ctx=ctx)
    cb, eb = orc.bin(model, cam, cfg16)
    np.testing.assert_array_equal(ca, cb)
    np.testing.assert_array_equal(ea, eb)


def test_render_empty_and_culled(orc, ctx):
    cam = make_camera(32)
    a = api.render(SplatModel(), cam, RenderConfig(), ctx=ctx)
    assert np.all(a.color == 1.0) and np.all(a.alpha == 0.0)
    behind = SplatModel(np.array([[0, 0, -5.0, -2, -2, -2, 1, 0, 0, 0, 0, 0.5, 0.5, 0.5]]))
    b = api.render(behind, cam, RenderConfig(background=(0.1, 0.2, 0.3)), ctx=ctx)
    np.testing.assert_allclose(b.color[..., 0], np.float32(0.1), rtol=0, atol=0)
    assert len(b.splat_order) == 0


def test_tiling_is_scheduling(ctx):
    model, cam, _ = SCENES[3]
    a = api.render(model, cam, RenderConfig(tile_size=16), ctx=ctx)
    b = api.render(model, cam, RenderConfig(tile_size=64), ctx=ctx)
    np.testing.assert_array_equal(a.color, b.color)


@pytest.mark.parametrize("lam", [0.0, 0.2, 1.0])
def test_loss_parity(orc, ctx, lam):
    rng = np.random.default_rng(3)
    a = rng.random((40, 36, 3)).astype(np.float32).astype(np.float64)
    b = np.clip(a + rng.normal(scale=0.05, size=a.shape), 0, 1).astype(np.float32).astype(np.float64)
    view = TrainView(make_camera(36), b, disc_mask(36, 40, 17.0, 20.0, 14.0))
    view.cam.height = 40
    la = api.masked_loss(a, view, lam, ctx=ctx)
    lb = orc.masked_loss(a, view, lam)
    assert abs(la.loss - lb.loss) <= 1e-6 * max(1.0, abs(lb.loss))
    scale = np.max(np.abs(lb.dL_dpixels))
    np.testing.assert_allclose(la.dL_dpixels, lb.dL_dpixels, rtol=1e-4, atol=1e-5 * scale)
    assert np.all(la.dL_dpixels[view.mask < 0.5] == 0.0)


def test_loss_vacuous_mask(ctx):
    view = TrainView(make_camera(32), np.full((32, 32, 3), 0.9), np.zeros((32, 32)))
    r = api.masked_loss(np.full((32, 32, 3), 0.1), view, 0.2, ctx=ctx)
    assert r.loss == 0.0 and np.all(r.dL_dpixels == 0.0)


def _loss_case(orc, model, cam, cfg, seed, mask):
    out = orc.render(model, cam, cfg)
    gt = offset_ground_truth(orc.render, model, cam, cfg, seed)
    view = TrainView(cam, gt, mask)
    return out, orc.masked_loss(out.color, view, 0.2)


@pytest.mark.parametrize("k", range(len(SCENES)))
def test_backward_parity(orc, ctx, k):
    model, cam, cfg = SCENES[k]
    out, lr = _loss_case(orc, model, cam, cfg, 7 + k,
                         disc_mask(cam.width, cam.height, cam.width * 0.45, cam.height * 0.5,
                                   cam.width * 0.35))
    ga = api.backward(model, cam, cfg, out, lr.dL_dpixels, ctx=ctx)
    gb = orc.backward(model, cam, cfg, out, lr.dL_dpixels)
    np.testing.assert_array_equal(ga.touch_count, gb.touch_count)
    assert_grads_close(ga.grads, gb.grads)


def test_backward_zero_in_zero_out(ctx):
    cam = make_camera(32)
    model = fp32_exact(random_scene(5, 4))
    out = api.render(model, cam, RenderConfig(), ctx=ctx)
    g = api.backward(model, cam, RenderConfig(), out, np.zeros((32, 32, 3)), ctx=ctx)
    assert np.all(g.grads == 0.0)


def test_backward_stale_forward(ctx):
    cam = make_camera(32)
    model = fp32_exact(random_scene(5, 2))
    out = api.render(model, cam, RenderConfig(), ctx=ctx)
    model.iteration += 1
    with pytest.raises(DsplatError, match="StaleForward"):
        api.backward(model, cam, RenderConfig(), out, np.zeros((32, 32, 3)), ctx=ctx)


def test_identity_rotation_gradients_exactly_zero(orc, ctx):
    model, cam, cfg = SCENES[7]  # isotropic, identity rotation
    out, lr = _loss_case(orc, model, cam, cfg, 3, full_mask(cam.width, cam.height))
    g = api.backward(model, cam, cfg, out, lr.dL_dpixels, ctx=ctx)
    assert np.all(g.grads[:, 6:10] == 0.0)


def test_adam_parity(orc, ctx):
    model = fp32_exact(random_scene(3, 64))
    rng = np.random.default_rng(5)
    G = (rng.normal(size=model.params.shape) * 1e-3).astype(np.float32).astype(np.float64)
    G[::7] = 0.0
    dm = api.DeviceModel(ctx, model)
    st = api.AdamState(dm)
    rates = GroupRates(1e-3, 5e-3, 1e-3, 5e-2, 5e-3)
    p = model.params.copy()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    step = 0
    for _ in range(3):
        st.step(api.GradientBuffer(G, None, None), rates)
        step = orc.adam_step(p, G, m, v, step, rates.as_tuple())
    out = dm.download()
    np.testing.assert_allclose(out.params, p, rtol=1e-5, atol=1e-7)
    mm, vv, s = dm.adam_state()
    assert s == 3
    np.testing.assert_allclose(mm, m, rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose(vv, v, rtol=1e-5, atol=1e-15)


def test_mask_bit_exact(orc, ctx):
    cam = make_camera(48)
    pts = random_cloud(9, 300, (-1.2, -1.2, -1.2), (1.2, 1.2, 1.2))
    for fp, dil in ((2.0, 2.0), (0.5, 0.0), (3.3, 1.7)):
        np.testing.assert_array_equal(api.render_mask(pts, cam, fp, dil, ctx=ctx),
                                      orc.render_mask(pts, cam, fp, dil))
    with pytest.raises(DsplatError, match="InvalidArgument"):
        api.render_mask(pts, cam, 0.2, 0.0, ctx=ctx)


def _train_setup(orc, n_views=3):
    cam0 = make_camera(48)
    target = fp32_exact(random_scene(24, 10))
    views = []
    for k in range(n_views):
        cam = make_camera(48)
        cam.position = (0.4 * k - 0.4, 0.1 * k, -3.0)
        gt = orc.render(target, cam, RenderConfig()).color
        views.append(TrainView(cam, gt, disc_mask(48, 48, 22.0 + k, 25.0, 19.0)))
    init = fp32_exact(random_scene(23, 10))
    return init, views, cam0


def test_train_first_step_parity(orc, ctx):
    init, views, _ = _train_setup(orc)
    cfg = TrainConfig(iterations=1, seed=9)
    a = api.train_partition_full(init, views, cfg, ctx=ctx, loss_trace=True)
    b = orc.train_partition_full(init, views, cfg, loss_trace=True)
    assert abs(a.final_loss - b.final_loss) <= 1e-6 * abs(b.final_loss)
    # after one step Adam moves every scalar by ~lr*sign(g): compare the steps
    step_a = a.model.params - init.params
    step_b = b.model.params - init.params
    assert_grads_close(step_a, step_b, rtol=1e-4, floor=1e-4)


def test_train_trajectory(orc, ctx):
    init, views, _ = _train_setup(orc)
    cfg = TrainConfig(iterations=30, seed=9, densify_interval=0)
    a = api.train_partition_full(init, views, cfg, ctx=ctx, loss_trace=True)
    b = orc.train_partition_full(init, views, cfg, loss_trace=True)
    np.testing.assert_allclose(a.loss_trace, b.loss_trace, rtol=2e-3)
    assert a.model.iteration == init.iteration + 30
    np.testing.assert_allclose(a.model.params, b.model.params, rtol=0, atol=5e-3)


def test_train_errors(ctx):
    model = fp32_exact(random_scene(3, 2))
    with pytest.raises(DsplatError, match="NoViews"):
        api.train_partition_full(model, [], TrainConfig(), ctx=ctx)
    view = TrainView(make_camera(32), np.full((32, 32, 3), 0.5), full_mask(32, 32))
    with pytest.raises(DsplatError, match="InvalidArgument"):
        api.train_partition_full(model, [view], TrainConfig(lr_mu=0.0), ctx=ctx)
    out = api.train_partition_full(model, [view], TrainConfig(iterations=0), ctx=ctx)
    np.testing.assert_array_equal(out.model.params, model.params)
