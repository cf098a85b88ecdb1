"""A full training run of the benched partition (config 2: 4M-Gaussian
Kingsnake partition, 403 views at 1024^2) with the reference's default
TrainConfig — densification every 100 steps until half way, lr_mu decay —
through dsg_train on one B200. Reports the loss trace, the model size after
each densification, the wall time and the held-out PSNR/SSIM before and
after, as JSON on stdout.

  python tools/long_run.py --iters 600 > gpurun_out/long_run.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=600)
    args = ap.parse_args()
    from bench import split_rig
    from paper_2509_12138_b200 import api, scenes
    from paper_2509_12138_b200.types import RenderConfig, TrainConfig
    ctx = api.Context(0)
    pts, cols, _ = scenes.kingsnake(scenes.SIZES["kingsnake"], seed=1, turns=6.0)
    nn = api.median_nn_spacing(pts, ctx=ctx)
    rig = scenes.rig_for_cloud(pts, 28, 16, 1024)
    train_idx, test_idx = split_rig(len(rig), 0.1, 1)
    rcfg = RenderConfig()
    gt = api.ground_truth_model(pts, cols, nn, 0.97, ctx=ctx)
    views = api.DeviceViews.synthesize(ctx, gt, rcfg, [rig[i] for i in train_idx], pts, True, 2.0, 2.0)
    dm = api.seed_gaussians(pts, cols, 3, ctx=ctx)
    test = [rig[i] for i in test_idx[:4]]

    def evaluate():
        ps = [api.eval_view(dm, gt, c, rcfg, ctx=ctx) for c in test]
        return float(np.mean([p for p, _ in ps])), float(np.mean([s for _, s in ps]))

    out = {"workload": "config 2 partition (4,000,000 Gaussians, 403 views at 1024^2)",
           "iters": args.iters, "train_config": "reference defaults (densify every 100 until 50%)"}
    out["before"] = dict(zip(("psnr", "ssim"), evaluate()))
    cfg = TrainConfig(iterations=args.iters, seed=1)
    n0 = dm.info()[0]
    t0 = time.perf_counter()
    fl, trace = api.train_device(dm, views, cfg, loss_trace=True)
    ctx.synchronize()
    wall = time.perf_counter() - t0
    out["wall_s"] = round(wall, 3)
    out["it_per_s"] = round(args.iters / wall, 2)
    out["final_loss"] = fl
    out["loss_every_50"] = [round(float(x), 6) for x in trace[::50]]
    out["model_size"] = {"start": int(n0), "end": int(dm.info()[0])}
    out["after"] = dict(zip(("psnr", "ssim"), evaluate()))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
