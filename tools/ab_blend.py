"""A/B harness for blend/binning changes: renders, losses and gradients of a
few config-2 views (Kingsnake 4M at 1024^2) with the library named by
DSG_LIB, saved to an npz; `--compare a.npz b.npz` reports the differences.

  DSG_LIB=.../libdsg_x.so python tools/ab_blend.py --out gpurun_out/x.npz
  python tools/ab_blend.py --compare gpurun_out/x.npz gpurun_out/y.npz
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(out, n, res, views, oracle_view=None):
    from paper_2509_12138_b200 import api, scenes
    from paper_2509_12138_b200.types import RenderConfig, TrainView
    ctx = api.Context(0)
    pts, cols, _ = scenes.kingsnake(n, seed=1)
    nn = api.median_nn_spacing(pts, ctx=ctx)
    rig = scenes.rig_for_cloud(pts, 28, 16, res)
    cams = [rig[i] for i in np.linspace(0, len(rig) - 1, views).astype(int)]
    gt = api.ground_truth_model(pts, cols, nn, 0.97, ctx=ctx)
    seeds = api.seed_gaussians(pts, cols, 3, ctx=ctx)
    rcfg = RenderConfig()
    res_ = {}
    for k, cam in enumerate(cams):
        g = api.render(gt, cam, rcfg, ctx=ctx)
        r = api.render(seeds, cam, rcfg, ctx=ctx)
        view = TrainView(cam, g.color, np.ones((cam.height, cam.width)))
        lo = api.masked_loss(r.color, view, 0.2, ctx=ctx)
        gb = api.backward(seeds, cam, rcfg, r, lo.dL_dpixels, ctx=ctx)
        res_[f"color{k}"] = r.color.astype(np.float32)
        res_[f"ncontrib{k}"] = r.per_pixel_contributor_count
        res_[f"loss{k}"] = np.array([lo.loss])
        res_[f"grads{k}"] = gb.grads.astype(np.float32)
        res_[f"touch{k}"] = gb.touch_count
    # a short training run on the same views (dsg_train: fused chain + Adam,
    # densification inside), then the trained parameters, moments and stats
    from paper_2509_12138_b200.types import TrainConfig
    dv = api.DeviceViews.synthesize(ctx, gt, rcfg, cams, pts, True, 2.0, 2.0)
    cfg = TrainConfig(iterations=2 * views, seed=1, densify_interval=3)
    fl, trace = api.train_device(seeds, dv, cfg, loss_trace=True)
    res_["train_params"] = seeds.download().params.astype(np.float32)
    m, v, st = seeds.adam_state()
    res_["train_m"], res_["train_v"] = m.astype(np.float32), v.astype(np.float32)
    res_["train_trace"] = trace
    if oracle_view is not None:
        # oracle contributor counts of one view (CPU, fp64 reference order)
        from oracle import Oracle
        o = Oracle().render(seeds.download(), cams[oracle_view], rcfg)
        res_["oracle_ncontrib"] = np.asarray(o.per_pixel_contributor_count)
        res_["oracle_color"] = o.color.astype(np.float32)
        res_["oracle_view"] = np.array([oracle_view])
    np.savez_compressed(out, **res_)
    print("saved", out)


def compare(a, b):
    A, B = np.load(a), np.load(b)
    worst = 0
    for k in sorted(A.files):
        x, y = A[k], B[k]
        same = np.array_equal(x, y)
        d = float(np.max(np.abs(x.astype(np.float64) - y.astype(np.float64)))) if x.size else 0.0
        ndiff = int(np.sum(x != y))
        print(f"{k:12s} identical={same} max|diff|={d:.3g} n_diff={ndiff}")
        worst = max(worst, ndiff)
    if "oracle_view" in B.files:
        v = int(B["oracle_view"][0])
        on = B["oracle_ncontrib"].reshape(A[f"ncontrib{v}"].shape)
        for name, X in (("A", A), ("B", B)):
            nc = X[f"ncontrib{v}"]
            bad = np.argwhere(nc != on)
            print(f"{name} vs oracle ncontrib view {v}: {len(bad)} pixels differ", bad[:10].tolist(),
                  [(int(nc[tuple(p)]), int(on[tuple(p)])) for p in bad[:10]])
    return worst


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    ap.add_argument("--n", type=int, default=4_000_000)
    ap.add_argument("--res", type=int, default=1024)
    ap.add_argument("--views", type=int, default=3)
    ap.add_argument("--compare", nargs=2)
    ap.add_argument("--oracle-view", type=int, default=None)
    a = ap.parse_args()
    if a.compare:
        compare(*a.compare)
    else:
        run(a.out, a.n, a.res, a.views, a.oracle_view)
