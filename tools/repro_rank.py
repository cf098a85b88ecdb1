"""Rebuild one rank's bench inputs on a single GPU and time the GT view
synthesis view by view (debugging slow or stuck ranks).

  python tools/repro_rank.py --world 4 --rank 0 [--views 20]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_12138_b200 import api, scenes  # noqa: E402
from paper_2509_12138_b200.types import RenderConfig  # noqa: E402
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=4)
ap.add_argument("--rank", type=int, default=0)
ap.add_argument("--n-per-gpu", type=int, default=4_000_000)
ap.add_argument("--views", type=int, default=1000)
ap.add_argument("--train", type=int, default=0)
ap.add_argument("--keys", action="store_true")
a = ap.parse_args()
ctx = api.Context(0)
n_total = a.n_per_gpu * a.world
pts, cols, _ = scenes.kingsnake(n_total, seed=1, turns=6.0 * a.world)
print("extent", pts.min(0), pts.max(0), flush=True)
nn = api.median_nn_spacing(pts, ctx=ctx)
parts = api.partition_cloud(pts, a.world, 3.0 * nn, ctx=ctx)
p = parts[a.rank]
idx = np.concatenate([p.owned_indices, p.ghost_indices]).astype(np.int64)
ppts, pcols = pts[idx], cols[idx]
print("partition", len(p.owned_indices), len(p.ghost_indices), "axis", p.cut_axis, p.cut_lo, p.cut_hi,
      "box", ppts.min(0), ppts.max(0), flush=True)
rig = scenes.rig_for_cloud(pts, 28, 16, 1024)
train_idx, _ = bench.split_rig(len(rig), 0.1, 1)
gt = api.ground_truth_model(ppts, pcols, nn, 0.97, ctx=ctx)
rc = RenderConfig()
for k, vi in enumerate(train_idx[: a.views]):
    cam = rig[vi]
    t0 = time.time()
    api.render(gt, cam, rc, ctx=ctx)
    st = api.frame_stats(ctx)
    dt = time.time() - t0
    if dt > 0.2 or k < 3:
        print(f"view {k} (rig {vi}) {dt:.3f}s {st} cam {cam.position}", flush=True)
        counts, _ = api.bin_splats(gt, cam, rc, ctx=ctx, capacity=1 << 24)
        c = np.sort(counts)[::-1]
        print("   busy tiles", int((c > 0).sum()), "top", c[:8].tolist(), "sum top16", int(c[:16].sum()))
print("done", flush=True)
if a.train:
    from paper_2509_12138_b200.types import TrainConfig
    cams = [rig[i] for i in train_idx[:16]]
    views = api.DeviceViews.synthesize(ctx, gt, rc, cams, ppts, True, 2.0, 2.0)
    seeds = api.seed_gaussians(ppts, pcols, 3, ctx=ctx)
    api.train_device(seeds, views, TrainConfig(iterations=3, seed=1))
    ctx.set_profiling(True)
    api.train_device(seeds, views, TrainConfig(iterations=a.train, seed=1))
    tot, st = ctx.last_timing()
    print("train ms/step", tot / a.train)
    for k, v in zip(api.STAGES, st):
        print(f"  {k:18s} {v / a.train:8.3f} ms")
if a.keys:
    from oracle import Oracle
    from paper_2509_12138_b200.types import TrainConfig
    seeds = api.seed_gaussians(ppts, pcols, 3, ctx=ctx)
    cam = rig[train_idx[0]]
    pr = Oracle().prepare(seeds.download(), cam, rc)
    d, ix = pr["depth"], pr["index"]
    lo, hi = d.min(), d.max()
    key = np.floor((d - lo) * (4294967295.0 / (hi - lo))).astype(np.uint64)
    order = np.lexsort((ix, key))
    ks, ds = key[order], d[order]
    same = ks[1:] == ks[:-1]
    inv = same & (ds[1:] < ds[:-1])
    # run lengths
    b = np.flatnonzero(np.concatenate([[True], ~same]))
    runs = np.diff(np.concatenate([b, [len(ks)]]))
    print("visible", len(d), "depth range", lo, hi, "quantum", (hi - lo) / 2**32)
    print("equal-key pairs", int(same.sum()), "inversions", int(inv.sum()), "max run", int(runs.max()),
          "runs>1", int((runs > 1).sum()), "exact ties", int((ds[1:] == ds[:-1]).sum()))
