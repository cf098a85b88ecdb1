"""TEST INFRASTRUCTURE ONLY — CPU checkers for the hot path.

Two interchangeable implementations of the same C ABI (oracle/orc_abi.h):

* ``Oracle()``     — liboracle.so, this repo's fp64 restatement (oracle.cpp)
* ``Reference()``  — _ref/libdsplat_ref.so, the unmodified reference headers
                     compiled here (only exists where /root/reference was
                     present at build time; the .so travels with the tree)

Both expose the reference API shape (render, masked_loss, backward, …) on the
host types of ``paper_2509_12138_b200.types``. Only tests/,
``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference legs may
import this package; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2509_12138_b200.types import (
    PARAMS, Camera, DsplatError, ErrorCode, GradientBuffer, LossResult, Partition, RenderConfig,
    RenderOutput, SplatModel, TrainConfig, TrainResult, TrainView)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdsplat_ref.so")


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and _ref when the reference headers exist)."""
    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class orc_camera(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("target", C.c_double * 3), ("up", C.c_double * 3),
                ("fov_y", C.c_double), ("width", C.c_int32), ("height", C.c_int32),
                ("near_plane", C.c_double), ("far_plane", C.c_double)]


class orc_render_cfg(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("_pad", C.c_int32), ("alpha_cutoff", C.c_double),
                ("sigma_cutoff", C.c_double), ("background", C.c_double * 3),
                ("transmittance_floor", C.c_double)]


class orc_train_cfg(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("lr_mu", C.c_double), ("lr_mu_decay", C.c_double),
                ("lr_scale", C.c_double), ("lr_rot", C.c_double), ("lr_opacity", C.c_double),
                ("lr_color", C.c_double), ("loss_lambda", C.c_double),
                ("densify_interval", C.c_int64), ("densify_grad_threshold", C.c_double),
                ("prune_opacity", C.c_double), ("densify_stop_fraction", C.c_double),
                ("split_scale_threshold", C.c_double), ("checkpoint_interval", C.c_int64),
                ("seed", C.c_uint64), ("render", orc_render_cfg), ("beta1", C.c_double),
                ("beta2", C.c_double), ("epsilon", C.c_double)]


def cam_struct(cam: Camera) -> orc_camera:
    c = orc_camera()
    c.position[:] = [float(v) for v in cam.position]
    c.target[:] = [float(v) for v in cam.target]
    c.up[:] = [float(v) for v in cam.up]
    c.fov_y = cam.fov_y
    c.width = cam.width
    c.height = cam.height
    c.near_plane = cam.near
    c.far_plane = cam.far
    return c


def cam_from_struct(c: orc_camera) -> Camera:
    return Camera(tuple(c.position), tuple(c.target), tuple(c.up), c.fov_y, c.width, c.height,
                  c.near_plane, c.far_plane)


def cfg_struct(cfg: RenderConfig) -> orc_render_cfg:
    c = orc_render_cfg()
    c.tile_size = cfg.tile_size
    c.alpha_cutoff = cfg.alpha_cutoff
    c.sigma_cutoff = cfg.sigma_cutoff
    c.background[:] = [float(v) for v in cfg.background]
    c.transmittance_floor = cfg.transmittance_floor
    return c


def train_struct(cfg: TrainConfig) -> orc_train_cfg:
    t = orc_train_cfg()
    for name in ("iterations", "lr_mu", "lr_mu_decay", "lr_scale", "lr_rot", "lr_opacity",
                 "lr_color", "loss_lambda", "densify_interval", "densify_grad_threshold",
                 "prune_opacity", "densify_stop_fraction", "split_scale_threshold",
                 "checkpoint_interval", "seed"):
        setattr(t, name, getattr(cfg, name))
    t.render = cfg_struct(cfg.render)
    t.beta1, t.beta2, t.epsilon = cfg.adam.beta1, cfg.adam.beta2, cfg.adam.epsilon
    return t


def _p(a, ct=C.c_double):
    return a.ctypes.data_as(C.POINTER(ct))


class _CpuImpl:
    """The reference API (render, masked_loss, backward, …) over one CPU .so."""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.lib.orc_last_error.restype = C.c_char_p
        self.lib.orc_impl_name.restype = C.c_char_p
        self.name = self.lib.orc_impl_name().decode()

    def _check(self, rc: int) -> None:
        if rc != 0:
            msg = self.lib.orc_last_error().decode()
            code = ErrorCode(rc - 1)
            raise DsplatError(code, msg.split(": ", 1)[1] if ": " in msg else msg)

    @staticmethod
    def _params(model):
        p = model.params if isinstance(model, SplatModel) else model
        return np.ascontiguousarray(p, dtype=np.float64).reshape(-1, PARAMS)

    # -- render path -------------------------------------------------------
    def prepare(self, model, cam: Camera, cfg: RenderConfig):
        P = self._params(model)
        n = P.shape[0]
        out = dict(index=np.zeros(n, np.int32), mean2d=np.zeros((n, 2)), inv_cov=np.zeros((n, 3)),
                   opacity=np.zeros(n), depth=np.zeros(n), rect=np.zeros((n, 4), np.int32))
        nv = C.c_int64()
        self._check(self.lib.orc_prepare(
            _p(P), C.c_int64(n), C.byref(cam_struct(cam)), C.byref(cfg_struct(cfg)), C.byref(nv),
            _p(out["index"], C.c_int32), _p(out["mean2d"]), _p(out["inv_cov"]),
            _p(out["opacity"]), _p(out["depth"]), _p(out["rect"], C.c_int32)))
        return {k: v[: nv.value] for k, v in out.items()}

    def bin(self, model, cam: Camera, cfg: RenderConfig, capacity: int = 1 << 22):
        P = self._params(model)
        tx = (cam.width + cfg.tile_size - 1) // cfg.tile_size
        ty = (cam.height + cfg.tile_size - 1) // cfg.tile_size
        counts = np.zeros(tx * ty, np.int32)
        entries = np.zeros(capacity, np.int32)
        ne = C.c_int64()
        self._check(self.lib.orc_bin(
            _p(P), C.c_int64(P.shape[0]), C.byref(cam_struct(cam)), C.byref(cfg_struct(cfg)),
            _p(counts, C.c_int32), _p(entries, C.c_int32), C.c_int64(capacity), C.byref(ne)))
        return counts, entries[: ne.value].copy()

    def render(self, model, cam: Camera, cfg: RenderConfig) -> RenderOutput:
        P = self._params(model)
        n = P.shape[0]
        h, w = cam.height, cam.width
        rgb = np.zeros((h, w, 3))
        alpha = np.zeros((h, w))
        nc = np.zeros((h, w), np.int32)
        order = np.zeros(max(n, 1), np.int32)
        no = C.c_int64()
        self._check(self.lib.orc_render(
            _p(P), C.c_int64(n), C.byref(cam_struct(cam)), C.byref(cfg_struct(cfg)), _p(rgb),
            _p(alpha), _p(nc, C.c_int32), _p(order, C.c_int32), C.byref(no)))
        it = model.iteration if isinstance(model, SplatModel) else 0
        return RenderOutput(rgb, alpha, nc, order[: no.value].copy(), it)

    def render_mask(self, points, cam: Camera, footprint_px: float, dilation_px: float):
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        mask = np.zeros((cam.height, cam.width))
        self._check(self.lib.orc_render_mask(
            _p(pts), C.c_int64(pts.shape[0]), C.byref(cam_struct(cam)), C.c_double(footprint_px),
            C.c_double(dilation_px), _p(mask)))
        return mask

    def masked_loss(self, rendered, view: TrainView, loss_lambda: float) -> LossResult:
        r = np.ascontiguousarray(rendered, dtype=np.float64)
        gt = np.ascontiguousarray(view.ground_truth, dtype=np.float64)
        m = np.ascontiguousarray(view.mask, dtype=np.float64)
        view.validate()
        if r.shape != gt.shape:
            raise DsplatError(ErrorCode.DimensionMismatch, "image dimensions differ")
        h, w = r.shape[:2]
        dL = np.zeros_like(r)
        loss = C.c_double()
        self._check(self.lib.orc_masked_loss(_p(r), _p(gt), _p(m), C.c_int32(w), C.c_int32(h),
                                             C.c_double(loss_lambda), C.byref(loss), _p(dL)))
        return LossResult(loss.value, dL)

    def ssim(self, a, b) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = C.c_double()
        self._check(self.lib.orc_ssim(_p(a), _p(b), C.c_int32(a.shape[1]), C.c_int32(a.shape[0]),
                                      C.byref(out)))
        return out.value

    def psnr(self, a, b) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64).ravel()
        b = np.ascontiguousarray(b, dtype=np.float64).ravel()
        out = C.c_double()
        self._check(self.lib.orc_psnr(_p(a), _p(b), C.c_int64(a.size), C.byref(out)))
        return out.value

    def backward(self, model: SplatModel, cam: Camera, cfg: RenderConfig, output: RenderOutput,
                 dL, shards: int = 1) -> GradientBuffer:
        P = self._params(model)
        n = P.shape[0]
        d = np.ascontiguousarray(dL, dtype=np.float64)
        if d.shape != (cam.height, cam.width, 3):
            raise DsplatError(ErrorCode.DimensionMismatch, "dL_dpixels must be RGB at camera resolution")
        G = np.zeros((n, PARAMS))
        dm = np.zeros((n, 2))
        tc = np.zeros(n, np.int32)
        self._check(self.lib.orc_backward(
            _p(P), C.c_int64(n), C.c_int64(model.iteration), C.c_int64(output.model_iteration),
            C.byref(cam_struct(cam)), C.byref(cfg_struct(cfg)), _p(d), C.c_int32(shards), _p(G),
            _p(dm), _p(tc, C.c_int32)))
        return GradientBuffer(G, dm, tc)

    def adam_step(self, params, grads, m, v, step: int, rates, adam=(0.9, 0.999, 1e-15)):
        """AdamState::step on explicit state; returns the new step count."""
        P = np.ascontiguousarray(params, dtype=np.float64)
        G = np.ascontiguousarray(grads, dtype=np.float64)
        st = C.c_int64(step)
        r = np.asarray(rates, dtype=np.float64)
        a = np.asarray(adam, dtype=np.float64)
        self._check(self.lib.orc_adam_step(_p(P), C.c_int64(P.shape[0]), _p(G), _p(m), _p(v),
                                           C.byref(st), _p(r), _p(a)))
        params[...] = P
        return st.value

    def train_partition_full(self, model: SplatModel, views, cfg: TrainConfig, shards: int = 1,
                             loss_trace: bool = False) -> TrainResult:
        P = self._params(model)
        n = P.shape[0]
        nv = len(views)
        if nv:
            h, w = views[0].cam.height, views[0].cam.width
            cams = (orc_camera * nv)(*[cam_struct(v.cam) for v in views])
            gts = np.ascontiguousarray(np.stack([v.ground_truth for v in views]), dtype=np.float64)
            masks = np.ascontiguousarray(np.stack([v.mask for v in views]), dtype=np.float64)
        else:
            cams = (orc_camera * 1)()
            gts = np.zeros(1)
            masks = np.zeros(1)
        cap = max(1, n) * 4 + 16
        out = np.zeros((cap, PARAMS))
        n_out = C.c_int64()
        fl = C.c_double()
        trace = np.zeros(max(1, cfg.iterations)) if loss_trace else None
        self._check(self.lib.orc_train(
            _p(P), C.c_int64(n), cams, _p(gts), _p(masks), C.c_int32(nv),
            C.byref(train_struct(cfg)), C.c_int32(shards), _p(out), C.c_int64(cap), C.byref(n_out),
            C.byref(fl), _p(trace) if trace is not None else None))
        res = TrainResult(SplatModel(out[: n_out.value].copy(), model.iteration + cfg.iterations,
                                     model.origin_partition), fl.value, n, n_out.value)
        if trace is not None:
            res.loss_trace = trace
        return res

    # -- float64 PLY (ply_io.hpp:89-221; oracle/_ref only) ---------------------
    def write_splat_ply(self, path: str, model: SplatModel):
        P = self._params(model)
        op = -1 if model.origin_partition is None else int(model.origin_partition)
        self._check(self.lib.orc_write_splat_ply(path.encode(), _p(P), C.c_int64(P.shape[0]),
                                                 C.c_int64(model.iteration), C.c_int32(op)))

    def read_splat_ply(self, path: str) -> SplatModel:
        n, it, op = C.c_int64(), C.c_int64(), C.c_int32()
        self._check(self.lib.orc_read_splat_ply(path.encode(), None, C.c_int64(0), C.byref(n),
                                                C.byref(it), C.byref(op)))
        P = np.zeros((max(n.value, 1), PARAMS))
        self._check(self.lib.orc_read_splat_ply(path.encode(), _p(P), C.c_int64(P.shape[0]),
                                                C.byref(n), C.byref(it), C.byref(op)))
        return SplatModel(P[: n.value], it.value, None if op.value < 0 else op.value)

    def write_cloud_ply(self, path: str, positions, normals, colors):
        pos, nrm, col = (np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)
                         for a in (positions, normals, colors))
        self._check(self.lib.orc_write_cloud_ply(path.encode(), _p(pos), _p(nrm), _p(col),
                                                 C.c_int64(pos.shape[0])))

    def train_partition(self, model, views, cfg, shards: int = 1) -> SplatModel:
        return self.train_partition_full(model, views, cfg, shards).model

    # -- partition / merge / rig -------------------------------------------
    def partition_cloud(self, positions, n: int, ghost_margin: float):
        pts = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        npts = pts.shape[0]
        ax = C.c_int32()
        lo = np.zeros(max(n, 1))
        hi = np.zeros(max(n, 1))
        box = np.zeros((max(n, 1), 6))
        oc = np.zeros(max(n, 1), np.int64)
        gc = np.zeros(max(n, 1), np.int64)
        cap = max(1, npts * max(n, 1))
        oi = np.zeros(cap, np.uint32)
        gi = np.zeros(cap, np.uint32)
        self._check(self.lib.orc_partition(
            _p(pts), C.c_int64(npts), C.c_int32(n), C.c_double(ghost_margin), C.byref(ax), _p(lo),
            _p(hi), _p(box), _p(oc, C.c_int64), _p(gc, C.c_int64), _p(oi, C.c_uint32),
            _p(gi, C.c_uint32), C.c_int64(cap)))
        parts = []
        o = g = 0
        for k in range(n):
            parts.append(Partition(k, ax.value, lo[k], hi[k], box[k].reshape(2, 3).copy(),
                                   ghost_margin, oi[o:o + oc[k]].copy(), gi[g:g + gc[k]].copy()))
            o += oc[k]
            g += gc[k]
        return parts

    def merge_keep(self, params_list, parts):
        """merge_models' per-splat keep flags over concatenated models."""
        counts = np.array([len(p) for p in params_list], np.int64)
        P = np.ascontiguousarray(np.concatenate([np.asarray(p).reshape(-1, PARAMS) for p in params_list]))
        keep = np.zeros(max(1, P.shape[0]), np.uint8)
        nk = C.c_int64()
        lo = np.array([p.cut_lo for p in parts])
        hi = np.array([p.cut_hi for p in parts])
        self._check(self.lib.orc_merge(_p(P), _p(counts, C.c_int64), C.c_int32(len(parts)),
                                       C.c_int32(parts[0].cut_axis), _p(lo), _p(hi),
                                       _p(keep, C.c_uint8), C.byref(nk)))
        return keep[: P.shape[0]].astype(bool)

    def build_orbital_cameras(self, center, radius, n_az, n_el, resolution, fov_y=0.9,
                              max_elevation=np.pi / 3.0):
        out = (orc_camera * max(1, n_az * n_el))()
        c = np.asarray(center, dtype=np.float64)
        self._check(self.lib.orc_orbital_cameras(
            _p(c), C.c_double(radius), C.c_int32(n_az), C.c_int32(n_el), C.c_int32(resolution),
            C.c_double(fov_y), C.c_double(max_elevation), out))
        return [cam_from_struct(out[i]) for i in range(n_az * n_el)]

    def split_rig(self, n_views: int, test_fraction: float, seed: int):
        tr = np.zeros(max(1, n_views), np.int32)
        te = np.zeros(max(1, n_views), np.int32)
        nt, ns = C.c_int64(), C.c_int64()
        self._check(self.lib.orc_split_rig(C.c_int64(n_views), C.c_double(test_fraction),
                                           C.c_uint64(seed), _p(tr, C.c_int32), C.byref(nt),
                                           _p(te, C.c_int32), C.byref(ns)))
        return tr[: nt.value].copy(), te[: ns.value].copy()

    # -- seeding -------------------------------------------------------------
    def knn_mean_distances(self, points, k: int):
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(pts.shape[0])
        self._check(self.lib.orc_knn_mean(_p(pts), C.c_int64(pts.shape[0]), C.c_int32(k), _p(out)))
        return out

    def median_nn_spacing(self, points) -> float:
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        out = C.c_double()
        self._check(self.lib.orc_median_nn(_p(pts), C.c_int64(pts.shape[0]), C.byref(out)))
        return out.value

    def seed_gaussians(self, points, colors, k: int = 3) -> SplatModel:
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        col = np.ascontiguousarray(colors, dtype=np.float64).reshape(-1, 3)
        P = np.zeros((pts.shape[0], PARAMS))
        self._check(self.lib.orc_seed_knn(_p(pts), _p(col), C.c_int64(pts.shape[0]), C.c_int32(k), _p(P)))
        return SplatModel(P)

    def ground_truth_model(self, points, colors, scale: float, opacity: float = 0.97) -> SplatModel:
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        col = np.ascontiguousarray(colors, dtype=np.float64).reshape(-1, 3)
        P = np.zeros((pts.shape[0], PARAMS))
        self._check(self.lib.orc_gt_model(_p(pts), _p(col), C.c_int64(pts.shape[0]),
                                          C.c_double(scale), C.c_double(opacity), _p(P)))
        return SplatModel(P)

    def rng_uniform(self, seed: int, count: int):
        out = np.zeros(count)
        self._check(self.lib.orc_rng_uniform(C.c_uint64(seed), C.c_int64(count), _p(out)))
        return out


_cache = {}


def Oracle() -> _CpuImpl:
    if "oracle" not in _cache:
        if not os.path.exists(ORACLE_SO):
            build()
        _cache["oracle"] = _CpuImpl(ORACLE_SO)
    return _cache["oracle"]


def Reference() -> _CpuImpl:
    """The reference headers compiled here; FileNotFoundError if absent."""
    if "ref" not in _cache:
        _cache["ref"] = _CpuImpl(REF_SO)
    return _cache["ref"]


def has_reference() -> bool:
    return os.path.exists(REF_SO)
