"""Parity of one training step at a benched / named configuration (TEST INFRASTRUCTURE).

Used by the `-m gpu` at-scale tests (tests/test_scale_parity.py) and by
bench.py's post-timing checker leg. The device path runs through the libdsg C
ABI (paper_2509_12138_b200.api); the checker is `oracle/_ref` (the reference
headers compiled unchanged) when present, else the pinned restatement.

Checks, with the north star's tolerances (BASELINE.json):
  * splat order (render.hpp:98-101) and per-tile lists at 16 px tiles
    (render.hpp:117-135): bit-exact
  * rendered RGB / alpha (render.hpp:160-205): max abs <= 1e-3
  * per-pixel contributor counts (render.hpp:183-199): exact
  * loss (loss.hpp:39-73): relative, reported
  * gradients (backward.hpp:184-332) from the same dL on both sides:
    |a-b| <= 1e-4 * max(|a|,|b|) + GRAD_FLOOR * max|b| per parameter group
  * touch counts: exact
  * post-Adam parameters (adam.hpp:55-101) from identical gradients: 1e-4
    relative (+1e-7 * group scale)
  * one full train iteration (trainer.hpp:173-207) each side: post-step
    parameters within 1e-4 relative wherever the reference gradient is above
    the floor; below it the sign of g is fp noise and, with epsilon = 1e-15,
    Adam moves the scalar by +-lr either way (the flips are counted)
"""
from __future__ import annotations

import time

import numpy as np

from paper_2509_12138_b200 import api
from paper_2509_12138_b200.types import GroupRates, RenderConfig, SplatModel, TrainConfig

IMG_TOL = 1e-3
GRAD_RTOL = 1e-4
GRAD_FLOOR = 1e-5
ADAM_RTOL = 1e-4
GROUPS = {"mu": slice(0, 3), "log_scale": slice(3, 6), "rot": slice(6, 10),
          "opacity": slice(10, 11), "color": slice(11, 14)}


def checker():
    """oracle/_ref when it was built here, else the pinned restatement."""
    from oracle import Oracle, Reference, has_reference
    return (Reference(), "reference") if has_reference() else (Oracle(), "port")


def grad_report(g_dev, g_ref, rtol=GRAD_RTOL, floor=GRAD_FLOOR):
    """Worst |a-b| / tol per group (<= 1 passes) and the max relative error
    over components above the floor."""
    out = {}
    for name, sl in GROUPS.items():
        a, b = g_dev[:, sl], g_ref[:, sl]
        scale = float(np.max(np.abs(b))) if b.size else 0.0
        tol = rtol * np.maximum(np.abs(a), np.abs(b)) + floor * scale
        err = np.abs(a - b)
        ratio = float(np.max(err / np.where(tol > 0, tol, 1.0))) if b.size else 0.0
        strong = np.abs(b) > floor * scale
        rel = float(np.max(err[strong] / np.abs(b[strong]))) if strong.any() else 0.0
        out[name] = {"worst_over_tol": ratio, "max_rel_above_floor": rel, "scale": scale,
                     "n_bad": int(np.sum(err > tol))}
        if ratio > 1.0:  # diagnostics: the worst components (splat, column, dev, ref)
            r = err / np.where(tol > 0, tol, 1.0)
            worst = np.argsort(r, axis=None)[-5:]
            out[name]["worst"] = [[int(i // r.shape[1]), int(i % r.shape[1]),
                                   float(a.flat[i]), float(b.flat[i])] for i in worst]
    return out


def forward_report(ctx, ref, model: SplatModel, cam, rcfg: RenderConfig):
    a = api.render(model, cam, rcfg, ctx=ctx)
    b = ref.render(model, cam, rcfg)
    cfg16 = RenderConfig(**{**rcfg.__dict__, "tile_size": 16})
    cap = 1 << 20
    while True:  # capacity: the device list length is only known after binning
        try:
            ca, ea = api.bin_splats(model, cam, cfg16, ctx=ctx, capacity=cap)
            break
        except Exception as e:  # noqa: BLE001
            if "capacity" not in str(e) or cap > (1 << 30):
                raise
            cap *= 4
    cb, eb = ref.bin(model, cam, cfg16, capacity=max(cap, len(ea) + 1))
    nc_mis = int(np.sum(a.per_pixel_contributor_count != b.per_pixel_contributor_count))
    return a, b, {
        "splat_order_bit_exact": bool(np.array_equal(a.splat_order, b.splat_order)),
        "n_visible": int(len(b.splat_order)),
        "tile_counts_bit_exact": bool(np.array_equal(ca, cb)),
        "tile_lists_bit_exact": bool(np.array_equal(ea, eb)),
        "n_tile_entries": int(len(eb)),
        "img_max_abs": float(np.max(np.abs(a.color - b.color))),
        "alpha_max_abs": float(np.max(np.abs(a.alpha - b.alpha))),
        "ncontrib_mismatch_px": nc_mis,
        "pixels": int(a.alpha.size),
    }


def step_parity(ctx, ref, model: SplatModel, view, tcfg: TrainConfig = None, shards: int = 0):
    """All checks above for `model` on `view` (a TrainView); returns a dict
    with an overall `pass` flag."""
    import os
    tcfg = tcfg or TrainConfig(iterations=1, seed=1)
    shards = shards or (os.cpu_count() or 1)
    rcfg = tcfg.render
    t0 = time.time()
    cam = view.cam
    a, b, rep = forward_report(ctx, ref, model, cam, rcfg)

    # loss: each side on its own image (the step's real inputs)
    la = api.masked_loss(a.color, view, tcfg.loss_lambda, ctx=ctx)
    lb = ref.masked_loss(b.color, view, tcfg.loss_lambda)
    rep["loss_dev"], rep["loss_ref"] = la.loss, lb.loss
    rep["loss_rel"] = abs(la.loss - lb.loss) / max(abs(lb.loss), 1e-300)

    # backward from the same dL (the reference's)
    ga = api.backward(model, cam, rcfg, a, lb.dL_dpixels, ctx=ctx)
    gb = ref.backward(model, cam, rcfg, b, lb.dL_dpixels, shards=shards)
    rep["grads"] = grad_report(ga.grads, gb.grads)
    rep["grad_worst_over_tol"] = max(v["worst_over_tol"] for v in rep["grads"].values())
    rep["grad_max_rel_above_floor"] = max(v["max_rel_above_floor"] for v in rep["grads"].values())
    rep["touch_count_exact"] = bool(np.array_equal(ga.touch_count, gb.touch_count))

    # Adam from identical gradients (the reference's)
    rates = GroupRates(tcfg.lr_mu, tcfg.lr_scale, tcfg.lr_rot, tcfg.lr_opacity, tcfg.lr_color)
    dm = api.DeviceModel(ctx, model)
    api.AdamState(dm).step(api.GradientBuffer(gb.grads, None, None), rates)
    pa = dm.download().params
    del dm
    pb = model.params.copy()
    m = np.zeros_like(pb)
    v = np.zeros_like(pb)
    ref.adam_step(pb, gb.grads, m, v, 0, rates.as_tuple())
    worst = 0.0
    for sl in GROUPS.values():
        x, y = pa[:, sl], pb[:, sl]
        tol = ADAM_RTOL * np.abs(y) + 1e-7 * max(float(np.max(np.abs(y))), 1e-30)
        worst = max(worst, float(np.max(np.abs(x - y) / tol)))
    rep["adam_worst_over_tol"] = worst

    # one full train iteration each side (render -> loss -> backward -> Adam)
    one = TrainConfig(**{**tcfg.__dict__, "iterations": 1})
    ta = api.train_partition_full(model, [view], one, ctx=ctx)
    t1 = time.perf_counter()
    tb = ref.train_partition_full(model, [view], one, shards=shards)
    rep["ref_train_iter_s"] = time.perf_counter() - t1
    da, db = ta.model.params - model.params, tb.model.params - model.params
    # L1 kinks: masked pixel channels where the two images sit on opposite
    # sides of the ground truth (|r - gt| below the image error), so
    # dL = l1w * sign(r - gt) (loss.hpp:58-66) differs by 2 * l1w between the
    # sides — a discontinuity of the reference itself, not a kernel error.
    # Splats compositing at those pixels are excluded from the post-step
    # check (the backward check above used the same dL on both sides).
    gt = np.asarray(view.ground_truth)
    kink = ((np.asarray(view.mask) >= 0.5)[..., None]
            & (np.sign(a.color - gt) != np.sign(b.color - gt)))
    affected = np.zeros(len(model), bool)
    if kink.any():
        gk = api.backward(model, cam, rcfg, a, kink.astype(np.float64), ctx=ctx)
        affected = np.any(gk.grads != 0.0, axis=1)
    rep["l1_kink_pixel_channels"] = int(kink.sum())
    dld, dlr = np.asarray(la.dL_dpixels), np.asarray(lb.dL_dpixels)
    off = ~kink if kink.ndim == dld.ndim else np.ones_like(dld, bool)
    rep["dL_max_rel_off_kinks"] = float(np.max(np.abs(dld - dlr)[off])
                                        / max(float(np.max(np.abs(dlr))), 1e-300)) if off.any() else 0.0
    rep["train_step_kink_splats_excluded"] = int(affected.sum())
    # Loss-conditioned components: each side's step starts from its own dL
    # (fp32 device loss on its image vs fp64 reference loss on its image;
    # the images differ by ~1e-6). The backward itself was checked above
    # with one dL, so the device gradient from its own dL (what dsg_train
    # uses) differs from the reference's only through that dL difference.
    # Where that moves a gradient beyond the gradient tolerance — components
    # that are near-total cancellations of many pixel terms — the Adam step
    # (lr * g / (|g| + 1e-15)) inherits it; those are excluded and counted.
    g_own = api.backward(model, cam, rcfg, a, la.dL_dpixels, ctx=ctx).grads
    loss_cond = np.zeros_like(g_own, bool)
    for sl in GROUPS.values():
        x, y = g_own[:, sl], gb.grads[:, sl]
        scale = float(np.max(np.abs(y))) if y.size else 0.0
        loss_cond[:, sl] = (np.abs(x - y) > GRAD_RTOL * np.maximum(np.abs(x), np.abs(y))
                            + GRAD_FLOOR * scale)
    rep["train_step_loss_conditioned_excluded"] = int(loss_cond.sum())
    # Step 1 of Adam maps a gradient g to lr * g / (|g| + eps) (eps = 1e-15),
    # whose slope lr * eps / (|g| + eps)^2 turns the gradient tolerance into
    # a step tolerance: with tol_g the tolerance at the reference gradient
    # and m = |g| - tol_g > 0 the smallest magnitude it admits, the step may
    # move by up to lr * eps * tol_g / m^2. Components with m <= 0 are below
    # the floor (their sign is not pinned by the gradient tolerance).
    eps = float(tcfg.adam.epsilon)
    flips, strong_bad = 0, 0
    for sl in GROUPS.values():
        gs = np.abs(gb.grads[:, sl])
        tol_g = GRAD_RTOL * gs + GRAD_FLOOR * gs.max()
        margin = gs - tol_g
        strong = (gs >= GRAD_FLOOR * gs.max()) & (margin > 0) if gs.max() > 0 \
            else np.zeros_like(gs, bool)
        strong &= ~affected[:, None]
        strong &= ~loss_cond[:, sl]
        x, y = da[:, sl], db[:, sl]
        with np.errstate(divide="ignore", over="ignore", invalid="ignore"):
            eps_term = np.abs(y) * eps * tol_g / np.maximum(margin, 1e-150) ** 2
        bad = (np.abs(x - y) > ADAM_RTOL * np.abs(y) + 1e-6 * max(float(np.abs(y).max()), 1e-30)
               + np.where(strong, eps_term, 0.0))
        strong_bad += int((bad & strong).sum())
        flips += int((bad & ~strong).sum())
        for i, c in np.argwhere(bad & strong)[:8]:  # diagnostics
            rep.setdefault("train_step_bad", []).append(
                [int(i), int(sl.start + c), float(x[i, c]), float(y[i, c]),
                 float(ga.grads[i, sl.start + c]), float(gb.grads[i, sl.start + c]),
                 float(gs[i, c] / gs.max())])
    rep["train_step_loss_rel"] = abs(ta.final_loss - tb.final_loss) / max(abs(tb.final_loss), 1e-300)
    rep["train_step_bad_above_floor"] = strong_bad
    rep["train_step_sign_flips_below_floor"] = flips
    rep["train_step_scalars"] = int(da.size)

    rep["pass"] = bool(rep["splat_order_bit_exact"] and rep["tile_counts_bit_exact"]
                       and rep["tile_lists_bit_exact"] and rep["img_max_abs"] <= IMG_TOL
                       and rep["alpha_max_abs"] <= IMG_TOL and rep["grad_worst_over_tol"] <= 1.0
                       and rep["touch_count_exact"] and rep["adam_worst_over_tol"] <= 1.0
                       and strong_bad == 0 and rep["loss_rel"] <= 1e-4
                       and rep["ncontrib_mismatch_px"] == 0)
    rep["gaussians"] = int(len(model))
    rep["resolution"] = [cam.width, cam.height]
    rep["checker_s"] = round(time.time() - t0, 1)
    return rep
