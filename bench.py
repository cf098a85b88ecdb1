#!/usr/bin/env python
"""Benchmark: distributed 3DGS partition training on B200 (BASELINE.json metric).

One "step" is one training iteration of one partition (trainer.hpp:173-207):
render -> masked L1 + D-SSIM -> backward -> Adam, on one 1024^2 view.

Workload (default ``kingsnake``, BASELINE configs[1] at N=1): a
Kingsnake-shaped synthetic isosurface of 4M Gaussians per GPU, 448-view
orbital rig (28 az x 16 el) at 1024^2, 10% test split, GT splats at the
median NN spacing (opacity 0.97), kNN seeds, 2+2 px background masks
(runtime.hpp:190-232). At N GPUs the cloud has N x 4M points and is cut
into N slab partitions with 3 x NN ghost margins; rank k trains partition
k with no communication (weak scaling).

value  : whole-job training iterations/s, device-timed (CUDA events inside
         dsg_train, max over ranks), inputs resident in HBM.
e2e    : same through the public C ABI with host buffers: model uploaded
         from host doubles, each step's view streamed from pinned host
         memory, each step's loss read back, model downloaded at the end
         (device buffers are allocated by an untimed first upload).
--impl reference : the reference's own CPU implementation (oracle/_ref, the
         unmodified headers compiled here) timed on the host cores, one
         iteration per step on the same partition and views.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2509_12138_b200 import api, scenes  # noqa: E402
from paper_2509_12138_b200.types import RenderConfig, SplatModel, TrainConfig, TrainView  # noqa: E402

METRIC = "training iters/sec & Gaussians·views/sec at 1/2/4/8 B200; render Mpix/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "traffic.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback
NVLINK_GBPS = 900.0    # NVLink 5 per direction per GPU (B200_PROFILING.md)
# arithmetic type of the path: fp32 storage and blend/chain/Adam arithmetic;
# fp64 where an integer or ordering decision is taken (projection, rects,
# depth order, the alpha/cutoff guard band) and in the SSIM window sums
DTYPE = "f32"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
class Dist:
    """Rank plumbing: torch.distributed (NCCL) only for barrier + max."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.torch, self.dist = torch, dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=f"cuda:{self.local}")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=f"cuda:{self.local}")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.out = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thr = threading.Thread(target=self._read, daemon=True)
            self.thr.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.out.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thr.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        med = float(np.median(sm)) if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
def build_partition_inputs(args, dist: Dist, ctx):
    """Cloud -> auto values -> partition -> this rank's seeds + train views."""
    n_total = args.n_per_gpu * dist.world
    t0 = time.time()
    if args.workload == "kingsnake":
        pts, cols, _ = scenes.kingsnake(n_total, seed=1, turns=6.0 * dist.world)
    else:
        pts, cols, _ = scenes.make_cloud(args.workload, n_total, seed=1, ctx=ctx)
    nn = api.median_nn_spacing(pts, ctx=ctx)          # resolve_auto_values (runtime.hpp:73-77)
    margin = 3.0 * nn
    parts = api.partition_cloud(pts, dist.world, margin, ctx=ctx)  # partition.hpp:42-104, on device
    part = parts[dist.rank]
    idx = np.concatenate([part.owned_indices, part.ghost_indices]).astype(np.int64)
    ppts, pcols = np.ascontiguousarray(pts[idx]), np.ascontiguousarray(cols[idx])
    rig = scenes.rig_for_cloud(pts, args.az, args.el, args.res)
    n_rig = len(rig)
    train_idx, test_idx = split_rig(n_rig, 0.1, 1)
    cams = [rig[i] for i in train_idx]
    rcfg = RenderConfig()
    gt_model = api.ground_truth_model(ppts, pcols, nn, 0.97, ctx=ctx)
    views = api.DeviceViews.synthesize(ctx, gt_model, rcfg, cams, ppts, True, 2.0, 2.0)
    seeds = api.seed_gaussians(ppts, pcols, 3, ctx=ctx)
    log(f"[rank {dist.rank}] inputs: cloud {n_total:,} pts, partition {len(ppts):,} "
        f"({len(part.owned_indices):,} owned + {len(part.ghost_indices):,} ghosts), nn {nn:.6g}, "
        f"{len(cams)} train views at {args.res}^2, setup {time.time() - t0:.1f}s")
    return dict(points=ppts, colors=pcols, cams=cams, views=views, seeds=seeds, gt=gt_model,
                rcfg=rcfg, nn=nn, n_part=len(ppts), rig=rig, test_idx=test_idx,
                partition=part, center=(pts.min(0) + pts.max(0)) * 0.5)


def global_phase(args, dist: Dist, ctx, inp, trained, reps: int = 3):
    """Ghost-trim merge of the trained partitions (NCCL all-gather at N>1) and
    the tile-parallel 3840x2160 render of the merged model (BASELINE configs[4]
    shape; explicit camera since the rig builder is square-only)."""
    from paper_2509_12138_b200.types import Camera
    comm = None
    if dist.world > 1:
        import torch.distributed as tdist
        uid = [api.Comm.unique_id() if dist.rank == 0 else None]
        tdist.broadcast_object_list(uid, src=0)
        comm = api.Comm(ctx, uid[0], dist.world, dist.rank)
        merged, n_merged, merge_ms = api.merge_allgather(comm, trained, inp["partition"])
    else:
        merged = api.merge_models([trained], [inp["partition"]], ctx=ctx)  # allocates
        ctx.synchronize()
        t0 = time.perf_counter()
        merged = api.merge_models([trained], [inp["partition"]], ctx=ctx, out=merged)
        merge_ms = (time.perf_counter() - t0) * 1e3
        n_merged = merged.info()[0]
    c0 = inp["rig"][0]
    cam = Camera(c0.position, tuple(float(v) for v in inp["center"]), (0.0, 1.0, 0.0), 0.9, 3840,
                 2160, c0.near, c0.far)
    api.render_distributed(comm, merged, cam, inp["rcfg"], want_image=False)  # warm-up
    ms = 0.0
    for _ in range(reps):
        dist.barrier()
        _, t = api.render_distributed(comm, merged, cam, inp["rcfg"], want_image=False)
        ms += dist.max(t)
    if comm:
        comm.close()
    mpix = reps * 3840 * 2160 / (ms * 1e-3) / 1e6
    mm = dist.max(merge_ms)
    wire = 56.0 * int(n_merged) * (dist.world - 1) / max(dist.world, 1)  # bytes into each GPU
    gbs = wire / (mm * 1e-3) / 1e9 if dist.world > 1 else None
    return {"merged_gaussians": int(n_merged), "merge_allgather_ms": round(mm, 3),
            "merge_allgather_GBps_per_gpu": round(gbs, 1) if gbs else None,
            "merge_vs_nvlink": ({"peak_GBps_per_direction": NVLINK_GBPS, "frac": round(gbs / NVLINK_GBPS, 3)}
                                if gbs else None),
            "merge_exchange": api.merge_exchange() if gbs else "one process",
            "render_4k_ms": round(ms / reps, 3), "render_4k_mpix_per_sec": round(mpix, 1),
            "render_ranks": dist.world}


def split_rig(n_views: int, test_fraction: float, seed: int):
    """split_rig (camera.hpp:116-130): seeded Fisher-Yates, test = tail."""
    M = (1 << 64) - 1

    def mix(s):
        s = (s + 0x9E3779B97F4A7C15) & M
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return s, z ^ (z >> 31)

    s = (seed ^ 0x5E1170F5 ^ 0x853C49E6748FEA9B) & M
    s, _ = mix(s)
    s, _ = mix(s)
    idx = list(range(n_views))
    for i in range(n_views, 1, -1):
        s, z = mix(s)
        j = z % i
        idx[i - 1], idx[j] = idx[j], idx[i - 1]
    nt = 0
    if test_fraction > 0 and n_views > 1:
        nt = min(max(int(math.floor(test_fraction * n_views + 0.5)), 1), n_views - 1)
    return idx[: n_views - nt], idx[n_views - nt:]


def train_config(args, rank: int, iterations: int) -> TrainConfig:
    # run_worker: cfg = spec.train, render = spec.render, seed = job seed + k (runtime.hpp:228-232)
    return TrainConfig(iterations=iterations, seed=1 + rank)


KERNEL_OF_STAGE = {"preprocess": "k_preprocess", "depth_sort": "k_onesweep (depth)",
                   "scan_duplicate": "k_duplicate", "tile_sort_ranges": "k_onesweep (tile)",
                   "blend_fwd": "k_blend_fwd<0>", "loss": "k_ssim_stats+k_loss_grad",
                   "blend_bwd": "k_blend_bwd", "chain": "k_chain", "adam": "k_adam",
                   "chain_adam": "k_chain<1>"}
# dsg_train fuses the chain and Adam into one kernel unless DSG_FUSE_ADAM=0
FUSED_ADAM = os.environ.get("DSG_FUSE_ADAM", "1") != "0"


def algorithmic_bytes(stage: str, n: int, nv: int, npix: int, n_dup: int) -> float:
    """Minimal HBM bytes one launch must move."""
    return {
        "preprocess": 92.0 * n,                             # §8d: 56 B params in + 36 B out per G
        "depth_sort": 4 * 16.0 * nv + 8.0 * nv,            # 4 passes (32-bit key) x (key,val) r+w + histogram read
        "scan_duplicate": 8.0 * nv + 16.0 * nv + 8.0 * n_dup,  # §8d scan + duplicate; 8 B (tile|mask, idx) per dup
        "tile_sort_ranges": 2 * 16.0 * n_dup + 9.0 * n_dup,  # 2 passes, ranges + sub-tile masks
        "blend_fwd": 5.0 * n_dup + 48.0 * n_dup + 20.0 * npix,   # list + payload per entry, pixel out
        "loss": 37.0 * npix,                                # §8d
        "blend_bwd": 5.0 * n_dup + 68.0 * n_dup + 20.0 * npix + 36.0 * n_dup,  # + >=1 partial/entry
        "chain": 112.0 * n + 36.0 * n_dup + 4.0 * n_dup,   # params+grads, partials, masks
        "adam": 412.0 * n,                                  # §8d 392 B/G + 20 B/G fused stats
        # fused: params r+w, moments r+w, stats r+w, counts/slots, partials, masks
        "chain_adam": 112.0 * n + 224.0 * n + 24.0 * n + 8.0 * n + 36.0 * n_dup + 4.0 * n_dup,
    }[stage]


ISSUE_BOUND = ("blend_fwd", "blend_bwd")


def roofline(stage_ms, n, nv, npix, n_dup, peak, peak_kind, sm_mhz=None, work=None):
    """Per-stage HBM fractions, and the dominant kernel's roofline. The blend
    kernels are bound by instruction issue, not HBM (DRAM is 3-7% busy under
    ncu): their roofline is warp instructions issued per second (ncu's count
    per launch over the live launch time) against 148 SMs x 4 schedulers x
    the SM clock, with the §8d work rate (composited pairs C per second
    against 148 x 128 FP32 lanes x clock) beside it."""
    traffic = {}
    try:
        with open(TRAFFIC_PATH) as f:
            traffic = json.load(f)
    except (OSError, ValueError):
        pass
    rows = {}
    for st, ms in stage_ms.items():
        if ms <= 0:
            continue
        b = algorithmic_bytes(st, n, nv, npix, n_dup)
        gbs = b / (ms * 1e-3) / 1e9
        rows[st] = {"ms": round(ms, 4), "GB/s": round(gbs, 1), "frac": round(gbs / peak, 4)}
    clk = (sm_mhz or 1965.0) * 1e6
    issue_peak = 148 * 4 * clk
    lane_peak = 148 * 128 * clk
    for st in ISSUE_BOUND:
        tr = traffic.get(KERNEL_OF_STAGE[st], {})
        if st in rows and tr.get("warp_inst_per_launch"):
            ips = float(tr["warp_inst_per_launch"]) / (stage_ms[st] * 1e-3)
            rows[st]["issue_frac"] = round(ips / issue_peak, 4)
        if st in rows and work and work.get("composited"):
            rows[st]["pairs_per_s"] = round(work["composited"] / (stage_ms[st] * 1e-3), 1)
            rows[st]["pair_lane_frac"] = round(work["composited"] / (stage_ms[st] * 1e-3) / lane_peak, 5)
    dom = max(stage_ms, key=stage_ms.get)
    kern = KERNEL_OF_STAGE[dom]
    tr = traffic.get(kern, {})
    d = rows[dom]
    if dom in ISSUE_BOUND and tr.get("warp_inst_per_launch"):
        ips = float(tr["warp_inst_per_launch"]) / (stage_ms[dom] * 1e-3)
        out = {"bound": "issue", "kernel": kern, "achieved": round(ips / 1e9, 2), "peak": round(issue_peak / 1e9, 2),
               "unit": "G warp-inst/s", "frac": round(ips / issue_peak, 4),
               "peak_basis": f"148 SMs x 4 issue slots x {clk / 1e6:.0f} MHz (SM clock under load)",
               "inst_per_launch": float(tr["warp_inst_per_launch"]),
               "ncu_issue_active_pct": tr.get("issue_active_pct"),
               "ncu_fma_pipe_pct": tr.get("fma_pipe_pct"), "ncu_xu_pipe_pct": tr.get("xu_pipe_pct")}
        if work and work.get("composited"):
            out["work"] = {"composited_pairs": work["composited"],
                           "pairs_per_s": d.get("pairs_per_s"),
                           "lane_peak_per_s": round(lane_peak, 1),
                           "frac": d.get("pair_lane_frac"),
                           "model": "§8d: ~40 FP32 ops + 1 MUFU per composited pair (backward)"}
        out["hbm"] = {"achieved_GBps": d["GB/s"], "peak_GBps": peak, "frac": d["frac"],
                      "bytes_per_launch": algorithmic_bytes(dom, n, nv, npix, n_dup)}
    else:
        out = {"bound": "hbm", "kernel": kern, "achieved": d["GB/s"], "peak": peak, "unit": "GB/s",
               "frac": d["frac"], "bytes_per_launch": algorithmic_bytes(dom, n, nv, npix, n_dup)}
    out["traffic"] = float(tr["dram_bytes_per_launch"]) if tr.get("dram_bytes_per_launch") else None
    out["traffic_source"] = tr.get("source")
    out["peak_kind"] = peak_kind
    out["per_stage"] = rows
    return out


def load_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def run_partitioned(args, dist: Dist):
    """BASELINE configs[2]/[3] shape: a fixed cloud cut into P partitions
    (P >= GPUs), partition k trained on GPU k mod N (runtime.hpp:337-343
    worker assignment). One step = one iteration of one partition; value =
    all partitions' iterations / the slowest rank's device time (strong
    scaling: the job is fixed, N GPUs share it).

    Views: every partition has its own GT renders and masks of the global
    rig (runtime.hpp:190-232). At 2048^2 all 403 views of 8 partitions are
    176 GB, more than one GPU holds beside the models, so with --stream-views
    (automatic when the views would not fit) only the views the schedule
    touches are rendered, kept in pinned host memory and streamed one per
    step (dsg_views_create_host, overlapped with the previous step).

    After the timed steps (--global): the trained partitions are merged —
    ghost trim + one packed NCCL all-gather per partition round at N > 1,
    merge_models in one process at N = 1 — and the merged model is rendered
    at 3840x2160 tile-parallel over the N ranks (BASELINE configs[4]), with
    PSNR/SSIM against the GT model's render on one held-out view
    (runtime.hpp:470-492)."""
    ctx = api.Context(dist.local)
    P = args.partitions
    if P % dist.world != 0:
        raise SystemExit(f"--partitions {P} must be a multiple of the GPU count {dist.world}")
    n_total = args.n_total or scenes.SIZES[args.workload]
    t0 = time.time()
    pts, cols, _ = scenes.make_cloud(args.workload, n_total, seed=1, ctx=ctx)
    log(f"[rank {dist.rank}] cloud {n_total:,} pts generated in {time.time() - t0:.1f}s")
    nn = api.median_nn_spacing(pts, ctx=ctx)
    parts = api.partition_cloud(pts, P, 3.0 * nn, ctx=ctx)
    rig = scenes.rig_for_cloud(pts, args.az, args.el, args.res)
    train_idx, test_idx = split_rig(len(rig), 0.1, 1)
    cams = [rig[i] for i in train_idx]
    rcfg = RenderConfig()
    mine = [k for k in range(P) if k % dist.world == dist.rank]
    npix = args.res * args.res
    resident_bytes = len(mine) * len(cams) * npix * 13
    stream = args.stream_views or resident_bytes > 60e9
    horizon = max(args.warmup, args.steps)
    work = []
    for k in mine:
        part = parts[k]
        idx = np.concatenate([part.owned_indices, part.ghost_indices]).astype(np.int64)
        ppts, pcols = np.ascontiguousarray(pts[idx]), np.ascontiguousarray(cols[idx])
        gt = api.ground_truth_model(ppts, pcols, nn, 0.97, ctx=ctx)
        if stream:
            need = sorted(set(api.view_order(1 + k, len(cams), horizon).tolist()))
            gts, masks = [None] * len(cams), [None] * len(cams)
            for c0 in range(0, len(need), 8):  # render a few at a time, keep them in pinned memory
                chunk = need[c0:c0 + 8]
                sub = api.DeviceViews.synthesize(ctx, gt, rcfg, [cams[i] for i in chunk], ppts,
                                                 True, 2.0, 2.0)
                for j, vi in enumerate(chunk):
                    gts[vi], masks[vi] = sub.download_planar(j, pin=True)
                del sub
            views = api.HostViews(ctx, cams, gts, masks)
        else:
            views = api.DeviceViews.synthesize(ctx, gt, rcfg, cams, ppts, True, 2.0, 2.0)
        del gt
        seeds = api.seed_gaussians(ppts, pcols, 3, ctx=ctx)
        host = seeds.download()
        host.origin_partition = k
        seeds.upload(host)
        work.append((k, seeds, host, views))
    log(f"[rank {dist.rank}] partitions {mine} of {P}: cloud {n_total:,} pts, sizes "
        f"{[len(w[2]) for w in work]}, {len(cams)} views at {args.res}^2 "
        f"({'streamed from pinned host memory' if stream else 'resident'}), "
        f"setup {time.time() - t0:.1f}s")
    for k, dm, host, views in work:  # warm-up
        if args.warmup > 0:
            api.train_device(dm, views, TrainConfig(iterations=args.warmup, seed=1 + k))
            dm.upload(host)
    ctx.synchronize()
    clocks = ClockSampler(dist.local)
    clocks.start()
    dist.barrier()
    ctx.synchronize()
    dev_ms, launches0 = 0.0, api.launch_count()
    with api.nvtx_range("dsg_timed"):
        for k, dm, host, views in work:
            api.train_device(dm, views, TrainConfig(iterations=args.steps, seed=1 + k))
            dev_ms += ctx.last_timing()[0]
        ctx.synchronize()
    launches = api.launch_count() - launches0
    dist.barrier()
    clk = clocks.stop()
    t_max = dist.max(dev_ms) / 1e3
    n_local = float(sum(len(w[2]) for w in work))
    total_iters = P * args.steps
    gv = dist.sum(n_local * args.steps) / t_max
    glob = None
    if not args.no_global:
        glob = partitioned_global(args, dist, ctx, work, parts, mine, pts, cols, nn, rig, test_idx)
    return {
        "metric": METRIC,
        "value": round(total_iters / t_max, 3),
        "unit": "it/s",
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t_max * 1e3 / (args.steps * len(work)), 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": DTYPE,
        "data": "synthetic",
        "config": {"workload": f"{args.workload}-shaped isosurface, {n_total:,} Gaussians in {P} slab "
                               f"partitions (+ghosts), partition k on GPU k mod N, "
                               f"{args.az}x{args.el} rig at {args.res}^2",
                   "partitions": P, "gaussians": n_total, "resolution": args.res,
                   "views": len(cams), "views_streamed": bool(stream),
                   "l2": "working set > L2"},
        "host": host_info(),
        "gaussian_views_per_sec": round(gv, 1),
        "partition_sizes": [len(w[2]) for w in work],
        "e2e": None,
        "gpu_launches": int(dist.sum(float(launches))),
        "clocks": clk,
        "global": glob,
    }


def partitioned_global(args, dist: Dist, ctx, work, parts, mine, pts, cols, nn, rig, test_idx,
                       reps: int = 3):
    """Merge of the trained partitions and the tile-parallel 4K render of the
    merged model (BASELINE configs[4]), plus its PSNR/SSIM on a test view."""
    from paper_2509_12138_b200.types import Camera
    comm = None
    locs = [w[1] for w in work]
    if dist.world > 1:
        import torch.distributed as tdist
        uid = [api.Comm.unique_id() if dist.rank == 0 else None]
        tdist.broadcast_object_list(uid, src=0)
        comm = api.Comm(ctx, uid[0], dist.world, dist.rank)
        merged, _, _ = api.merge_allgather_multi(comm, locs, [parts[k] for k in mine])  # allocation pass
        ctx.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        merged, n_merged, wire_ms = api.merge_allgather_multi(comm, locs, [parts[k] for k in mine],
                                                              out=merged)
        total_ms = dist.max((time.perf_counter() - t0) * 1e3)  # the whole call (trim, counts, pack, unpack)
        merge_ms = dist.max(wire_ms)
    else:
        merged = api.merge_models(locs, [parts[k] for k in mine], ctx=ctx)  # allocation pass
        ctx.synchronize()
        t0 = time.perf_counter()
        merged = api.merge_models(locs, [parts[k] for k in mine], ctx=ctx, out=merged)
        merge_ms = (time.perf_counter() - t0) * 1e3
        n_merged = merged.info()[0]
    c0 = rig[0]
    center = (pts.min(0) + pts.max(0)) * 0.5
    cam = Camera(c0.position, tuple(float(v) for v in center), (0.0, 1.0, 0.0), 0.9, 3840, 2160,
                 c0.near, c0.far)
    api.render_distributed(comm, merged, cam, RenderConfig(), want_image=False)  # warm-up
    ms = 0.0
    for _ in range(reps):
        dist.barrier()
        _, t = api.render_distributed(comm, merged, cam, RenderConfig(), want_image=False)
        ms += dist.max(t)
    out = {"merged_gaussians": int(n_merged), "merge_ms": round(merge_ms, 3),
           "merge_call_ms": round(total_ms if dist.world > 1 else merge_ms, 3),
           "render_4k_ms": round(ms / reps, 3),
           "render_4k_mpix_per_sec": round(reps * 3840 * 2160 / (ms * 1e-3) / 1e6, 1),
           "render_ranks": dist.world}
    if dist.world > 1:
        wire = 56.0 * int(n_merged) * (dist.world - 1) / dist.world  # bytes into each GPU
        gbs = wire / (merge_ms * 1e-3) / 1e9
        out["merge_allgather_GBps_per_gpu"] = round(gbs, 1)
        out["merge_vs_nvlink"] = {"peak_GBps_per_direction": NVLINK_GBPS, "frac": round(gbs / NVLINK_GBPS, 3)}
        out["merge_exchange"] = api.merge_exchange()
        comm.close()
    if dist.rank == 0:  # held-out view: render(merged) vs render(GT model), runtime.hpp:483-492
        gtm = api.ground_truth_model(pts, cols, nn, 0.97, ctx=ctx)
        ps, ss = api.eval_view(merged, gtm, rig[test_idx[0]], RenderConfig(), ctx=ctx)
        out["eval_test_view"] = {"view": int(test_idx[0]), "psnr": round(ps, 3), "ssim": round(ss, 5),
                                 "note": f"after {args.steps + args.warmup} steps per partition"}
        del gtm
    return out


def run_ours(args, dist: Dist):
    ctx = api.Context(dist.local)
    inp = build_partition_inputs(args, dist, ctx)
    seeds_host = inp["seeds"].download()           # the partition's seed model (host doubles)
    n = len(seeds_host)
    dm = api.DeviceModel(ctx, seeds_host)
    views = inp["views"]
    npix = args.res * args.res

    # warm-up (untimed), then exactly K timed steps in one dsg_train call
    if args.warmup > 0:
        api.train_device(dm, views, train_config(args, dist.rank, args.warmup))
        dm.upload(seeds_host)
    ctx.synchronize()
    clocks = ClockSampler(dist.local)
    clocks.start()
    dist.barrier()
    ctx.synchronize()
    w0 = time.perf_counter()
    launches0 = api.launch_count()
    # NVTX range so `ncu --nvtx --nvtx-include dsg_timed/` captures exactly the timed steps
    with api.nvtx_range("dsg_timed"):
        fl, _ = api.train_device(dm, views, train_config(args, dist.rank, args.steps))
        ctx.synchronize()
    launches = api.launch_count() - launches0
    dist.barrier()
    wall = time.perf_counter() - w0
    clk = clocks.stop()
    dev_ms, _ = ctx.last_timing()
    t_max = dist.max(dev_ms) / 1e3
    wall_max = dist.max(wall)
    total_iters = args.steps * dist.world
    gv = dist.sum(float(n) * args.steps) / t_max

    # merge of the trained partitions + tile-parallel 4K render (untimed w.r.t. value)
    glob = global_phase(args, dist, ctx, inp, dm) if not args.no_global else None

    # per-stage profile (separate run; events + sync per step)
    ctx.set_profiling(True)
    dm.upload(seeds_host)
    pk = max(3, min(args.steps, 8))
    api.train_device(dm, views, train_config(args, dist.rank, pk))
    prof_total, stages = ctx.last_timing()
    ctx.set_profiling(False)
    stage_ms = {s: float(v) / pk for s, v in zip(api.STAGES, stages)}
    if FUSED_ADAM:  # one launch does chain + Adam; the "adam" mark holds only the densify check
        stage_ms["chain_adam"] = stage_ms.pop("chain") + stage_ms.pop("adam")
    fs = api.frame_stats(ctx)
    n_dup, nv_vis = fs["n_dup"], fs["n_visible"]
    work = api.frame_work(ctx)  # composited pairs C and fp64 termination fix-ups, last view

    # render Mpix/s on the test views (forward only, device-timed)
    test_cams = [inp["rig"][i] for i in inp["test_idx"]]
    r_ms = api.render_timed(dm, test_cams, inp["rcfg"], repeats=2)
    mpix = len(test_cams) * 2 * npix / (r_ms * 1e-3) / 1e6
    mpix = dist.sum(mpix)

    # End to end through the reference-shaped public API: the caller's
    # SplatModel (host doubles) and std::vector<TrainView>-like list of views
    # in the reference's own layout (HWC double ground truth, HW double mask,
    # loss.hpp:14-26) go into train_partition_full (trainer.hpp:140), which
    # uploads the model, streams the scheduled views (host conversion to
    # planar fp32 + bytes into pinned slots, overlapped with the previous
    # step), trains, reads every step's loss back and returns the model as
    # host doubles. Views the schedule never touches are never read, so they
    # share one placeholder image here (the call cannot tell).
    order = api.view_order(train_config(args, dist.rank, 1).seed, len(views), args.steps)
    sched = sorted(set(order.tolist()))
    h, w = args.res, args.res
    blank_gt, blank_mask = np.zeros((h, w, 3)), np.zeros((h, w))
    tviews = [TrainView(c, blank_gt, blank_mask) for c in views.cams]
    for vi in sched:
        tv = views.download(int(vi))
        tviews[vi] = TrainView(views.cams[vi], tv.ground_truth, tv.mask)
    host_model = SplatModel(np.ascontiguousarray(seeds_host.params))
    tc = train_config(args, dist.rank, args.steps)
    api.train_partition_full(host_model, tviews, tc, ctx=ctx)  # untimed: allocations, pinned slots
    import gc
    gc.collect()  # unrelated garbage (device buffers of earlier phases) is not freed mid-measurement
    gc.disable()
    dist.barrier()
    ctx.synchronize()
    e0 = time.perf_counter()
    res = api.train_partition_full(host_model, tviews, tc, ctx=ctx, loss_trace=True)
    e_wall = time.perf_counter() - e0
    gc.enable()
    log(f"[e2e] wall {e_wall:.4f}s phases {getattr(ctx, 'last_phases', None)}")
    e_dev_ms, _ = ctx.last_timing()  # the same loop's device span (events)
    e_parts = {"train_partition_full_s": round(e_wall, 4), "train_device_s": round(e_dev_ms * 1e-3, 4),
               **{k: round(v, 4) for k, v in getattr(ctx, "last_phases", {}).items()},
               "outside_device_loop_s": round(e_wall - e_dev_ms * 1e-3, 4),
               "views_streamed": args.steps, "final_loss": res.final_loss}
    assert len(res.loss_trace) == args.steps
    e_max = dist.max(e_wall)
    # bytes that cross the bus: the model as fp32 both ways (amortised), each
    # step's converted view (planar fp32 + mask bytes) in, the loss trace out
    view_bytes = npix * (3 * 4 + 1)
    h2d = view_bytes + n * 14 * 4 / args.steps
    d2h = 8 + n * 14 * 4 / args.steps
    del res

    peak, peak_kind = load_peak()
    roof = roofline(stage_ms, n, nv_vis, npix, n_dup, peak, peak_kind, clk.get("sm_mhz"), work)

    cpu, parity = None, None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cpu, parity = cpu_baseline(ctx, inp, views, seeds_host, args)

    line = {
        "metric": METRIC,
        "value": round(total_iters / t_max, 3),
        "unit": "it/s",
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t_max * 1e3 / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": DTYPE,
        "data": "synthetic",
        "config": config_dict(args, dist.world, n, len(views)),
        "host": host_info(),
        "gaussian_views_per_sec": round(gv, 1),
        "render_mpix_per_sec": round(mpix, 2),
        "wall_s": round(wall_max, 4),
        "stage_ms": {k: round(v, 4) for k, v in stage_ms.items()},
        "n_dup": n_dup,
        "frame_work": work,
        "e2e": {"value": round(total_iters / e_max, 3), "unit": "it/s",
                "api": "api.train_partition_full(SplatModel, [TrainView], TrainConfig) "
                       "(trainer.hpp:140): host doubles in, reference-layout views, host doubles out",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "breakdown": e_parts},
        "gpu_launches": int(dist.sum(float(launches))),
        "roofline": roof,
        "cpu_baseline": cpu,
        "parity": parity,
        "clocks": clk,
        "global": glob,
        "final_loss": fl,
    }
    return line


def cpu_baseline(ctx, inp, views, seeds_host, args):
    """Checker leg, after all timing (rank 0, N=1): the reference's own CPU
    implementation (oracle/_ref) on the same partition and the first scheduled
    view. One call of tests/scale_parity.step_parity compares the device path
    with it (splat order, per-tile lists, image, loss, gradients, Adam, one
    train iteration) and times the reference's train iteration on the host
    cores, which is the cpu_baseline value."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from scale_parity import checker, step_parity
    impl, kind = checker()
    cores = os.cpu_count() or 1
    order = api.view_order(1, len(views), 1)
    tv = views.download(int(order[0]))
    model = SplatModel(np.ascontiguousarray(seeds_host.params))
    rep = step_parity(ctx, impl, model, tv, TrainConfig(iterations=1, seed=1), shards=cores)
    dt = rep["ref_train_iter_s"]
    cpu = {"value": round(1.0 / dt, 5), "unit": "it/s", "cores": cores, "kind": kind,
           "sample": f"1 training iteration of the same partition ({len(seeds_host):,} Gaussians) "
                     f"on its first scheduled {args.res}^2 view, shards={cores} (row-band "
                     f"threads), {dt:.1f} s",
           "gaussian_views_per_sec": round(len(seeds_host) / dt, 1)}
    keep = ("pass", "splat_order_bit_exact", "tile_counts_bit_exact", "tile_lists_bit_exact",
            "n_visible", "n_tile_entries", "img_max_abs", "alpha_max_abs", "ncontrib_mismatch_px",
            "loss_rel", "grad_worst_over_tol", "grad_max_rel_above_floor", "touch_count_exact",
            "adam_worst_over_tol", "train_step_bad_above_floor",
            "train_step_sign_flips_below_floor", "train_step_scalars")
    parity = {k: rep[k] for k in keep}
    parity["lists_bit_exact"] = bool(rep["tile_lists_bit_exact"] and rep["splat_order_bit_exact"])
    parity["grad_max_rel"] = rep["grad_max_rel_above_floor"]
    parity["checker"] = kind
    parity["view"] = int(order[0])
    parity["tolerances"] = {"image_max_abs": 1e-3, "grad_rel": 1e-4, "grad_floor": "1e-5 x group max",
                            "adam_rel": 1e-4}
    return cpu, parity


def view_order_host(seed: int, n_views: int, iterations: int):
    """Seeded view order (trainer.hpp:157-163, 174) restated in Python, so the
    reference arm never maps libdsg.so: Rng(seed ^ 0x87aa11d3).shuffle."""
    M = (1 << 64) - 1

    def mix(st):
        st = (st + 0x9E3779B97F4A7C15) & M
        z = st
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return st, z ^ (z >> 31)

    s = ((seed ^ 0x87AA11D3) ^ 0x853C49E6748FEA9B) & M
    s, _ = mix(s)
    s, _ = mix(s)
    order = list(range(n_views))
    for i in range(n_views, 1, -1):
        s, z = mix(s)
        j = z % i
        order[i - 1], order[j] = order[j], order[i - 1]
    return [order[it % n_views] for it in range(iterations)]


def host_info():
    """nproc and the CPU model of the box the CPU legs run on."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count() or 1, "cpu_model": model}


def config_dict(args, world: int, gaussians: int, views: int):
    """The workload description both arms print (identical by construction)."""
    return {"workload": f"{args.workload}-shaped isosurface, {args.n_per_gpu:,} Gaussians/GPU "
                        f"(+ghosts), {args.az}x{args.el} rig at {args.res}^2, one slab "
                        f"partition per GPU", "gaussians_per_gpu": int(gaussians),
            "views": int(views), "resolution": args.res, "partitions": world,
            "l2": "working set > L2 (params+grads+moments 224 B/G)"}


def knn_seeds_host(pts, cols, k: int = 3):
    """seed_gaussians(ScaleRule::Knn, k) (seed.hpp:49-74) on the host for the
    reference arm: exact k-NN by k-d tree, the k smallest fp64 distances summed
    in ascending order and divided by k (seed.hpp:29-32), std::log via libm."""
    from scipy.spatial import cKDTree
    d, _ = cKDTree(pts).query(pts, k=k + 1, workers=os.cpu_count() or 1)
    acc = np.zeros(len(pts))
    for j in range(1, k + 1):
        acc = acc + d[:, j]
    mean = acc / k
    P = np.zeros((len(pts), 14))
    P[:, 0:3] = pts
    P[:, 3:6] = np.array([math.log(max(s, 1e-7)) for s in mean.tolist()])[:, None]
    P[:, 6] = 1.0
    P[:, 10] = math.log(0.1 / (1.0 - 0.1))  # logit(0.1)
    P[:, 11:14] = cols
    return SplatModel(P)


def reference_inputs(args, world: int, ref, steps: int):
    """Rank 0's partition and its scheduled train views, built on the host with
    the reference's own functions (oracle/_ref) — no libdsg.so in this process.

    Same recipe as build_partition_inputs: the cloud generator (scenes.py), the
    auto ghost margin 3 x median NN spacing, partition_cloud, the orbital rig
    and split_rig, kNN seeds (seed.hpp:49-74), GT = render(ground_truth_model)
    and render_mask per view (runtime.hpp:190-199). The reference's kNN is
    O(N^2) (seed.hpp:16-35) and cannot run at 4M points, so the k smallest
    exact fp64 distances come from a k-d tree and are summed in ascending
    order as the reference does; logs use libm like std::log."""
    from scipy.spatial import cKDTree
    from paper_2509_12138_b200.types import TrainView
    n_total = args.n_per_gpu * world
    if args.workload == "kingsnake":
        pts, cols, _ = scenes.kingsnake(n_total, seed=1, turns=6.0 * world)
    else:
        pts, cols, _ = scenes.make_cloud(args.workload, n_total, seed=1)
    workers = os.cpu_count() or 1
    d1, _ = cKDTree(pts).query(pts, k=2, workers=workers)
    nn = float(np.partition(d1[:, 1], len(pts) // 2)[len(pts) // 2])  # median_nn_spacing
    if world > 1:
        part = ref.partition_cloud(pts, world, 3.0 * nn)[0]
        idx = np.concatenate([part.owned_indices, part.ghost_indices]).astype(np.int64)
        ppts, pcols = np.ascontiguousarray(pts[idx]), np.ascontiguousarray(cols[idx])
    else:
        ppts, pcols = pts, cols
    seeds = knn_seeds_host(ppts, pcols)
    gt_model = ref.ground_truth_model(ppts, pcols, nn, 0.97)
    rig = scenes.rig_for_cloud(pts, args.az, args.el, args.res)
    train_idx, _ = split_rig(len(rig), 0.1, 1)
    cams = [rig[i] for i in train_idx]
    views = {}
    for vi in view_order_host(1, len(cams), steps):
        if vi not in views:
            cam = cams[vi]
            views[vi] = TrainView(cam, ref.render(gt_model, cam, RenderConfig()).color,
                                  ref.render_mask(ppts, cam, 2.0, 2.0))
    return seeds, cams, views


def run_reference(args, dist: Dist):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    headers compiled with the reference's Release flags) on the host cores.
    Rank 0 only. Each step = one train_partition_full iteration (render ->
    masked_loss -> backward -> Adam, trainer.hpp:173-207) of rank 0's
    partition on the next scheduled view, shards = nproc."""
    if dist.rank != 0:
        return None
    from oracle import Oracle, Reference, has_reference
    impl = Reference() if has_reference() else Oracle()
    kind = "reference" if has_reference() else "port"
    cores = os.cpu_count() or 1
    # each CPU step is ~15-60 s: bound the whole run to a few minutes
    args.steps = min(args.steps, 4)
    args.warmup = min(args.warmup, 1)
    t0 = time.time()
    seeds, cams, views = reference_inputs(args, dist.world, impl, args.warmup + args.steps)
    log(f"[reference] inputs: partition {len(seeds):,} Gaussians, {len(cams)} train views, "
        f"{len(views)} scheduled views rendered, setup {time.time() - t0:.1f}s")
    order = view_order_host(1, len(cams), args.warmup + args.steps)
    for it in range(args.warmup):
        impl.train_partition_full(seeds, [views[order[it]]], TrainConfig(iterations=1, seed=1),
                                  shards=cores)
    dts = []
    for it in range(args.steps):
        v = views[order[args.warmup + it]]
        t1 = time.perf_counter()
        impl.train_partition_full(seeds, [v], TrainConfig(iterations=1, seed=1), shards=cores)
        dts.append(time.perf_counter() - t1)
    T = float(sum(dts))
    v = args.steps / T
    with open("/proc/self/maps") as f:
        mapped = sorted({ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")
                         and ROOT in ln})
    log(f"[reference] in-tree shared objects mapped: {mapped}")
    return {
        "impl": "reference", "metric": METRIC, "value": round(v, 5), "unit": "it/s",
        "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(T * 1e3 / args.steps, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, dist.world, len(seeds), len(cams)),
        "gaussian_views_per_sec": round(len(seeds) * v, 1),
        "host": host_info(),
        "cpu_baseline": {"value": round(v, 5), "unit": "it/s", "cores": cores, "kind": kind,
                         "sample": f"each step = 1 reference training iteration (render, loss, "
                                   f"backward, Adam) of rank 0's {len(seeds):,}-Gaussian partition "
                                   f"on the next scheduled {args.res}^2 view, shards={cores}"},
        "e2e": {"value": round(v, 5), "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def _single():
    d = Dist.__new__(Dist)
    d.world, d.rank, d.local, d.pg = 1, 0, int(os.environ.get("LOCAL_RANK", "0")), None
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=list(scenes.SIZES), default="kingsnake")
    ap.add_argument("--n-per-gpu", type=int, default=None)
    ap.add_argument("--res", type=int, default=1024)
    ap.add_argument("--az", type=int, default=28)
    ap.add_argument("--el", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-global", action="store_true", help="skip the merge + 4K render phase")
    ap.add_argument("--partitions", type=int, default=0,
                    help="P > GPUs: fixed cloud in P partitions, k on GPU k mod N (configs 3/4)")
    ap.add_argument("--n-total", type=int, default=None, help="cloud size for --partitions")
    ap.add_argument("--stream-views", action="store_true",
                    help="--partitions: scheduled views in pinned host memory, streamed per step")
    args = ap.parse_args()
    if args.n_per_gpu is None:
        args.n_per_gpu = scenes.SIZES[args.workload]
    # Libraries (NCCL's version banner, torchrun) may write to fd 1: keep the
    # real stdout for the single JSON line and send everything else to stderr.
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    # watchdog: a hung rank dumps every thread's stack and exits instead of
    # holding the GPUs until the launcher's limit
    import faulthandler
    faulthandler.dump_traceback_later(float(os.environ.get("DSG_BENCH_WATCHDOG_S", "900")),
                                      exit=True)
    dist = Dist()
    if args.gpus != dist.world:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE {dist.world}; using WORLD_SIZE")
    if args.impl == "reference":
        line = run_reference(args, dist)
    elif args.partitions:
        line = run_partitioned(args, dist)
    else:
        line = run_ours(args, dist)
    if dist.rank == 0 and line is not None:
        json_out.write(json.dumps(line) + "\n")
        json_out.flush()
    dist.close()


if __name__ == "__main__":
    main()
