"""§8f #4: float64 PLY (ply_io.hpp:89-221) and PSNR/SSIM (metrics.hpp:20-38).

CPU tests: the point-cloud PLY (host code in libdsg) is byte-identical to the
reference's write_cloud_ply and round-trips bit-exactly. GPU tests: a device
model's PLY is byte-identical to the reference's write_splat_ply of the same
values and loads back bit-exactly; PSNR/SSIM on the device match the
reference's metrics.
"""
import os

import numpy as np
import pytest

from oracle import Reference, has_reference
from paper_2509_12138_b200 import api, scenes
from paper_2509_12138_b200.types import DsplatError, RenderConfig, SplatModel
from util import fp32_exact, random_scene
from util import test_camera as make_camera

needs_ref = pytest.mark.skipif(not has_reference(), reason="oracle/_ref not built")


@needs_ref
def test_cloud_ply_bytes_and_round_trip(tmp_path):
    pts, cols, nrm = scenes.sphere(5000)
    pts[7] = [-0.0, 1e-300, -1e300]  # odd values survive a float64 container
    a, b = str(tmp_path / "a.ply"), str(tmp_path / "b.ply")
    api.write_cloud_ply(a, pts, nrm, cols)
    Reference().write_cloud_ply(b, pts, nrm, cols)
    assert open(a, "rb").read() == open(b, "rb").read()
    p2, n2, c2 = api.read_cloud_ply(a)
    for x, y in ((p2, pts), (n2, nrm), (c2, cols)):
        assert x.tobytes() == np.ascontiguousarray(y).tobytes()


def test_cloud_ply_errors(tmp_path):
    bad = tmp_path / "bad.ply"
    bad.write_bytes(b"PLY\nend_header\n")
    with pytest.raises(DsplatError, match="not a ply file"):
        api.read_cloud_ply(str(bad))
    bad.write_bytes(b"ply\nformat ascii 1.0\nelement vertex 0\nend_header\n")
    with pytest.raises(DsplatError, match="binary_little_endian"):
        api.read_cloud_ply(str(bad))
    bad.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 1\n"
                    b"property float x\nend_header\n")
    with pytest.raises(DsplatError, match="expected double properties, got float"):
        api.read_cloud_ply(str(bad))
    good = tmp_path / "good.ply"
    api.write_cloud_ply(str(good), np.zeros((4, 3)), np.zeros((4, 3)), np.zeros((4, 3)))
    bad.write_bytes(good.read_bytes()[:-8])
    with pytest.raises(DsplatError, match="ply payload truncated"):
        api.read_cloud_ply(str(bad))
    with pytest.raises(DsplatError, match="IoError"):
        api.read_cloud_ply(str(tmp_path / "missing.ply"))


@pytest.mark.gpu
@needs_ref
def test_splat_ply_matches_reference(tmp_path):
    ctx = api.Context(0)
    model = fp32_exact(random_scene(5, 3000))
    model.iteration, model.origin_partition = 123, 4
    dm = api.DeviceModel(ctx, model)
    a, b = str(tmp_path / "a.ply"), str(tmp_path / "b.ply")
    dm.save_ply(a)
    Reference().write_splat_ply(b, model)  # model is fp32-exact: the device holds the same values
    assert open(a, "rb").read() == open(b, "rb").read()
    back = api.read_splat_ply(a, ctx=ctx)
    np.testing.assert_array_equal(back.params, model.params)
    assert back.iteration == 123 and back.origin_partition == 4
    r = Reference().read_splat_ply(a)
    np.testing.assert_array_equal(r.params, model.params)
    # no origin comment when the model has none
    dm2 = api.DeviceModel(ctx, SplatModel(model.params[:5], 7))
    dm2.save_ply(a)
    Reference().write_splat_ply(b, SplatModel(model.params[:5], 7))
    assert open(a, "rb").read() == open(b, "rb").read()
    bad = tmp_path / "bad.ply"
    api.write_cloud_ply(str(bad), np.zeros((2, 3)), np.zeros((2, 3)), np.zeros((2, 3)))
    with pytest.raises(DsplatError, match="splat ply must have 14 properties"):
        api.read_splat_ply(str(bad), ctx=ctx)


@pytest.mark.gpu
def test_image_metrics_match_reference():
    from oracle import Oracle
    orc = Reference() if has_reference() else Oracle()
    ctx = api.Context(0)
    rng = np.random.default_rng(4)
    a = rng.random((37, 45, 3)).astype(np.float32).astype(np.float64)
    b = np.clip(a + rng.normal(scale=0.03, size=a.shape), 0, 1).astype(np.float32).astype(np.float64)
    ps, ss = api.image_metrics(a, b, ctx=ctx)
    assert abs(ps - orc.psnr(a, b)) <= 1e-9 * abs(ps)
    assert abs(ss - orc.ssim(a, b)) <= 1e-12
    assert api.image_metrics(a, a, ctx=ctx)[0] == 99.0  # kPsnrCap
    with pytest.raises(DsplatError, match="TooSmall"):
        api.image_metrics(a[:10, :10], b[:10, :10], ctx=ctx)


@pytest.mark.gpu
def test_eval_view_matches_reference():
    """runtime.hpp:483-492: psnr/ssim of render(merged) vs render(gt)."""
    from oracle import Oracle
    orc = Reference() if has_reference() else Oracle()
    ctx = api.Context(0)
    model = fp32_exact(random_scene(8, 200))
    truth = fp32_exact(random_scene(9, 200))
    cam = make_camera(64)
    cfg = RenderConfig()
    ps, ss = api.eval_view(model, truth, cam, cfg, ctx=ctx)
    ra, rb = orc.render(model, cam, cfg).color, orc.render(truth, cam, cfg).color
    assert abs(ps - orc.psnr(ra, rb)) <= 1e-4 * abs(ps)
    assert abs(ss - orc.ssim(ra, rb)) <= 1e-5
