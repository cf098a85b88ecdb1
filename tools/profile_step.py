"""Profiling driver: config-2 partition (Kingsnake-shaped, 4M, 1024^2) with a
small rig, then a few training steps — short enough to run under ncu.

  python tools/profile_step.py [--n 4000000] [--res 1024] [--iters 3]
Launch order: 7 GT renders (k_blend_fwd), then per step one k_blend_fwd and
one k_blend_bwd.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_12138_b200 import api, scenes  # noqa: E402
from paper_2509_12138_b200.types import RenderConfig, TrainConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4_000_000)
ap.add_argument("--res", type=int, default=1024)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--workload", default="kingsnake")
args = ap.parse_args()

ctx = api.Context(0)
pts, cols, _ = scenes.make_cloud(args.workload, args.n, seed=1)
nn = api.median_nn_spacing(pts, ctx=ctx)
rig = scenes.rig_for_cloud(pts, 28, 16, args.res)
cams = [rig[i] for i in (5, 60, 117, 200, 251, 333, 401)]
gt = api.ground_truth_model(pts, cols, nn, 0.97, ctx=ctx)
views = api.DeviceViews.synthesize(ctx, gt, RenderConfig(), cams, pts, True, 2.0, 2.0)
seeds = api.seed_gaussians(pts, cols, 3, ctx=ctx)
api.train_device(seeds, views, TrainConfig(iterations=3, seed=1))  # warm-up: allocations
seeds.upload(seeds.download())
ctx.set_profiling(True)
api.train_device(seeds, views, TrainConfig(iterations=args.iters, seed=1))
tot, st = ctx.last_timing()
print("total ms/step", tot / args.iters)
for k, v in zip(api.STAGES, st):
    print(f"  {k:18s} {v / args.iters:8.3f} ms")
print(api.frame_stats(ctx))
