"""Small end-to-end exercise of every device path for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):

  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_step.py

render (incl. long split lists and the fp64 termination fix-up), bin,
masked loss, backward, Adam, a short training run with densification,
partition, merge, views synthesis, PLY and metrics — on scenes small enough
that the sanitizer's slowdown stays in minutes."""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2509_12138_b200 import api, scenes  # noqa: E402
from paper_2509_12138_b200.types import RenderConfig, SplatModel, TrainConfig, TrainView  # noqa: E402
from util import fp32_exact, random_scene  # noqa: E402
from util import test_camera as make_camera  # noqa: E402


def main():
    ctx = api.Context(0)
    cfg = RenderConfig()
    cam = make_camera(64)
    m = fp32_exact(random_scene(99, 300))
    m.params[:, 3:6] -= 1.5
    r = api.render(m, cam, cfg, ctx=ctx)
    api.bin_splats(m, cam, RenderConfig(tile_size=16), ctx=ctx)
    gt = api.render(fp32_exact(random_scene(98, 300)), cam, cfg, ctx=ctx).color
    view = TrainView(cam, gt, np.ones((64, 64)))
    lr = api.masked_loss(r.color, view, 0.2, ctx=ctx)
    api.backward(m, cam, cfg, r, lr.dL_dpixels, ctx=ctx)
    # a tile list long enough for the split forward and segment checkpoints
    rng = np.random.default_rng(11)
    n = 40000
    p = np.zeros((n, 14))
    p[:, 0] = rng.uniform(-0.02, 0.02, n)
    p[:, 1] = rng.uniform(-0.02, 0.02, n)
    p[:, 2] = rng.uniform(-0.3, 0.3, n)
    p[:, 3:6] = np.log(rng.uniform(0.001, 0.004, (n, 3)))
    p[:, 6] = 1.0
    p[:, 10] = rng.uniform(-2.5, 1.5, n)
    p[:, 11:14] = rng.uniform(0.1, 0.9, (n, 3))
    big = fp32_exact(SplatModel(p))
    rb = api.render(big, cam, cfg, ctx=ctx)
    api.backward(big, cam, cfg, rb, rng.normal(size=rb.color.shape) * 0.01, ctx=ctx)
    print("frame work", api.frame_work(ctx))
    tc = TrainConfig(iterations=12, seed=3, densify_interval=5, densify_grad_threshold=1e-6,
                     split_scale_threshold=0.05)
    api.train_partition_full(m, [view], tc, ctx=ctx)
    pts, cols, _ = scenes.sphere(20000)
    parts = api.partition_cloud(pts, 3, 0.01, ctx=ctx)
    seeds = [api.seed_gaussians(pts[np.concatenate([q.owned_indices, q.ghost_indices])],
                                cols[np.concatenate([q.owned_indices, q.ghost_indices])], 3, ctx=ctx)
             for q in parts]
    merged = api.merge_models(seeds, parts, ctx=ctx)
    cams = scenes.rig_for_cloud(pts, 4, 2, 64)[:3]
    gtm = api.ground_truth_model(pts, cols, 0.01, 0.97, ctx=ctx)
    views = api.DeviceViews.synthesize(ctx, gtm, cfg, cams, pts, True, 2.0, 2.0)
    api.train_device(seeds[0], views, TrainConfig(iterations=3, seed=2))
    api.render_distributed(None, merged, cams[0], cfg)
    api.eval_view(merged, gtm, cams[1], cfg, ctx=ctx)
    with tempfile.TemporaryDirectory() as d:
        merged.save_ply(os.path.join(d, "m.ply"))
        api.read_splat_ply(os.path.join(d, "m.ply"), ctx=ctx)
    api.heightfield_cloud("rt", 50000, 1, ctx=ctx)
    ctx.synchronize()
    print("SANITIZE_STEP_OK")


if __name__ == "__main__":
    main()
