"""Generate tests/golden/*.npz from the reference itself (TEST INFRASTRUCTURE).

Runs the unmodified reference (oracle/_ref/libdsplat_ref.so, built by
oracle/Makefile from /root/reference/proj/include) on small fixed inputs and
stores inputs and outputs, so the oracle restatement and the device path can
be checked against the reference's own numbers where the reference is not
available (the GPU box carries these files, not /root/reference).

    python tests/golden/make_golden.py      # rewrites tests/golden/golden.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import Reference  # noqa: E402
from paper_2509_12138_b200.types import (GroupRates, RenderConfig, SplatModel, TrainConfig,  # noqa: E402
                                         TrainView)
from util import disc_mask, fp32_exact, random_cloud, random_scene  # noqa: E402
from util import test_camera as make_camera  # noqa: E402

CASES = [  # (scene seed, splats, resolution, log-scale shift)
    (21, 12, 48, 0.0),
    (55, 40, 64, -0.5),
    (99, 300, 64, -1.5),
]


def main():
    ref = Reference()
    out = {}
    cfg = RenderConfig()
    for i, (seed, n, res, shift) in enumerate(CASES):
        m = random_scene(seed, n)
        m.params[:, 3:6] += shift
        m = fp32_exact(m)
        cam = make_camera(res)
        r = ref.render(m, cam, cfg)
        counts, entries = ref.bin(m, cam, RenderConfig(tile_size=16))
        gt = fp32_exact(random_scene(seed + 1, n))
        g_img = ref.render(gt, cam, cfg).color
        view = TrainView(cam, g_img, disc_mask(res, res, res * 0.5, res * 0.5, res * 0.4))
        lr = ref.masked_loss(r.color, view, 0.2)
        gb = ref.backward(m, cam, cfg, r, lr.dL_dpixels)
        out[f"c{i}_params"] = m.params
        out[f"c{i}_res"] = np.array([res])
        out[f"c{i}_color"] = r.color
        out[f"c{i}_alpha"] = r.alpha
        out[f"c{i}_ncontrib"] = r.per_pixel_contributor_count
        out[f"c{i}_order"] = r.splat_order
        out[f"c{i}_tile_counts"] = counts
        out[f"c{i}_tile_entries"] = entries
        out[f"c{i}_gt"] = g_img
        out[f"c{i}_mask"] = view.mask
        out[f"c{i}_loss"] = np.array([lr.loss])
        out[f"c{i}_dL"] = lr.dL_dpixels
        out[f"c{i}_grads"] = gb.grads
        out[f"c{i}_touch"] = gb.touch_count
        # one Adam step from those gradients, then a 5-step training run
        p = m.params.copy()
        mm, vv = np.zeros_like(p), np.zeros_like(p)
        ref.adam_step(p, gb.grads, mm, vv, 0, GroupRates(1e-3, 5e-3, 1e-3, 5e-2, 5e-3).as_tuple())
        out[f"c{i}_adam_params"] = p
        tr = ref.train_partition_full(m, [view], TrainConfig(iterations=5, seed=7), loss_trace=True)
        out[f"c{i}_train_params"] = tr.model.params
        out[f"c{i}_train_trace"] = tr.loss_trace
    pts = random_cloud(9, 2000)
    out["part_points"] = pts
    for nparts, margin in ((3, 0.1), (5, 0.0)):
        parts = ref.partition_cloud(pts, nparts, margin)
        for k, p in enumerate(parts):
            out[f"part{nparts}_{k}_owned"] = p.owned_indices
            out[f"part{nparts}_{k}_ghost"] = p.ghost_indices
            out[f"part{nparts}_{k}_cuts"] = np.array([p.cut_lo, p.cut_hi, p.cut_axis])
    mcam = make_camera(48)
    out["mask_points"] = pts[:300]
    out["mask_2_2"] = ref.render_mask(pts[:300], mcam, 2.0, 2.0)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
