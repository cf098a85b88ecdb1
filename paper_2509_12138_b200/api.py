"""Reference-shaped host API over libdsg.so (include/dsg.h) via ctypes.

Same names, argument meaning and error behaviour as the reference C++ API
(proj/include/dsplat): ``render`` (render.hpp:160), ``render_mask``
(render.hpp:210), ``masked_loss`` (loss.hpp:39), ``backward``
(backward.hpp:184), ``AdamState.step`` (adam.hpp:55),
``train_partition_full`` / ``train_partition`` (trainer.hpp:140, 214).
Every call runs on the B200 through the C ABI; if libdsg.so is missing or no
sm_100 device is present the call raises — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .types import (PARAMS, AdamConfig, Camera, DsplatError, ErrorCode, GradientBuffer, GroupRates,
                    LossResult, RenderConfig, RenderOutput, SplatModel, TrainConfig, TrainResult,
                    TrainView)

HERE = os.path.dirname(os.path.abspath(__file__))
# DSG_LIB selects an alternative in-tree build (A/B kernel experiments only).
LIB_PATH = os.environ.get("DSG_LIB") or os.path.join(HERE, "libdsg.so")


class dsg_camera(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("target", C.c_double * 3), ("up", C.c_double * 3),
                ("fov_y", C.c_double), ("width", C.c_int32), ("height", C.c_int32),
                ("near_plane", C.c_double), ("far_plane", C.c_double)]


class dsg_render_config(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("_pad", C.c_int32), ("alpha_cutoff", C.c_double),
                ("sigma_cutoff", C.c_double), ("background", C.c_double * 3),
                ("transmittance_floor", C.c_double)]


class dsg_adam_config(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("epsilon", C.c_double)]


class dsg_group_rates(C.Structure):
    _fields_ = [("mu", C.c_double), ("log_scale", C.c_double), ("rot", C.c_double),
                ("opacity", C.c_double), ("color", C.c_double)]


class dsg_train_config(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("lr_mu", C.c_double), ("lr_mu_decay", C.c_double),
                ("lr_scale", C.c_double), ("lr_rot", C.c_double), ("lr_opacity", C.c_double),
                ("lr_color", C.c_double), ("loss_lambda", C.c_double),
                ("densify_interval", C.c_int64), ("densify_grad_threshold", C.c_double),
                ("prune_opacity", C.c_double), ("densify_stop_fraction", C.c_double),
                ("split_scale_threshold", C.c_double), ("checkpoint_interval", C.c_int64),
                ("seed", C.c_uint64), ("render", dsg_render_config), ("adam", dsg_adam_config)]


PROGRESS_FN = C.CFUNCTYPE(None, C.c_int64, C.c_double, C.c_void_p)
CHECKPOINT_FN = C.CFUNCTYPE(None, C.c_int64, C.c_double, C.c_void_p, C.c_void_p)

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load libdsg.so (raises if it was not built — no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"libdsg.so not built at {LIB_PATH}; run __graft_entry__.build()")
            L = C.CDLL(LIB_PATH)
            L.dsg_last_error.restype = C.c_char_p
            _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().dsg_last_error().decode()
        code = ErrorCode(rc - 1)
        raise DsplatError(code, msg.split(": ", 1)[1] if ": " in msg else msg)


def _p(a, ct=C.c_double):
    return None if a is None else a.ctypes.data_as(C.POINTER(ct))


def cam_struct(cam: Camera) -> dsg_camera:
    c = dsg_camera()
    c.position[:] = [float(v) for v in cam.position]
    c.target[:] = [float(v) for v in cam.target]
    c.up[:] = [float(v) for v in cam.up]
    c.fov_y = cam.fov_y
    c.width = cam.width
    c.height = cam.height
    c.near_plane = cam.near
    c.far_plane = cam.far
    return c


def cfg_struct(cfg: RenderConfig) -> dsg_render_config:
    c = dsg_render_config()
    c.tile_size = cfg.tile_size
    c.alpha_cutoff = cfg.alpha_cutoff
    c.sigma_cutoff = cfg.sigma_cutoff
    c.background[:] = [float(v) for v in cfg.background]
    c.transmittance_floor = cfg.transmittance_floor
    return c


def train_struct(cfg: TrainConfig) -> dsg_train_config:
    t = dsg_train_config()
    for name in ("iterations", "lr_mu", "lr_mu_decay", "lr_scale", "lr_rot", "lr_opacity",
                 "lr_color", "loss_lambda", "densify_interval", "densify_grad_threshold",
                 "prune_opacity", "densify_stop_fraction", "split_scale_threshold",
                 "checkpoint_interval", "seed"):
        setattr(t, name, getattr(cfg, name))
    t.render = cfg_struct(cfg.render)
    t.adam = dsg_adam_config(cfg.adam.beta1, cfg.adam.beta2, cfg.adam.epsilon)
    return t


class Context:
    """One CUDA device + stream (dsg_ctx). Not thread-safe."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        _check(lib().dsg_ctx_create(C.c_int32(device), C.byref(self.h)))
        self.device = device

    def close(self):
        if self.h:
            lib().dsg_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(lib().dsg_ctx_synchronize(self.h))

    def scratch_model(self, model: SplatModel) -> "DeviceModel":
        """A device model owned by this context, reused across calls of the
        host-in/host-out entry points (its buffers only grow), so repeated
        train_partition_full calls do not re-allocate ~224 B per Gaussian."""
        if getattr(self, "_scratch", None) is None:
            self._scratch = DeviceModel(self)
        self._scratch.upload(model)
        return self._scratch

    def set_profiling(self, on: bool):
        _check(lib().dsg_set_profiling(self.h, C.c_int32(1 if on else 0)))

    def last_timing(self):
        tot = C.c_double()
        st = np.zeros(len(STAGES))
        _check(lib().dsg_last_timing(self.h, C.byref(tot), _p(st)))
        return tot.value, st


STAGES = ("preprocess", "depth_sort", "scan_duplicate", "tile_sort_ranges", "blend_fwd", "loss",
          "blend_bwd", "chain", "adam")


class DeviceModel:
    """A splat model resident on the device (dsg_model)."""

    def __init__(self, ctx: Context, model: SplatModel = None):
        self.ctx = ctx
        self.h = C.c_void_p()
        _check(lib().dsg_model_create(ctx.h, C.byref(self.h)))
        if model is not None:
            self.upload(model)

    def __del__(self):
        try:
            if self.h:
                lib().dsg_model_destroy(self.h)
        except Exception:
            pass

    def upload(self, model: SplatModel):
        P = np.ascontiguousarray(model.params, dtype=np.float64)
        op = -1 if model.origin_partition is None else int(model.origin_partition)
        _check(lib().dsg_model_upload(self.ctx.h, self.h, _p(P), C.c_int64(P.shape[0]),
                                      C.c_int64(model.iteration), C.c_int32(op)))

    def info(self):
        n, it, st = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().dsg_model_info(self.h, C.byref(n), C.byref(it), C.byref(st)))
        return n.value, it.value, st.value

    def download(self) -> SplatModel:
        n, _, _ = self.info()
        P = np.empty((max(n, 1), PARAMS))
        nn, it, op = C.c_int64(), C.c_int64(), C.c_int32()
        _check(lib().dsg_model_download(self.ctx.h, self.h, _p(P), C.c_int64(P.shape[0]),
                                        C.byref(nn), C.byref(it), C.byref(op)))
        return SplatModel(P[: nn.value], it.value, None if op.value < 0 else op.value)

    def save_ply(self, path: str):
        """write_splat_ply (ply_io.hpp:89-119) straight from the device store."""
        _check(lib().dsg_model_save_ply(self.ctx.h, self.h, os.fsencode(path)))

    def load_ply(self, path: str):
        """read_splat_ply (ply_io.hpp:121-158) into this device model."""
        _check(lib().dsg_model_load_ply(self.ctx.h, self.h, os.fsencode(path)))

    def adam_state(self):
        n, _, _ = self.info()
        m = np.zeros((max(n, 1), PARAMS))
        v = np.zeros((max(n, 1), PARAMS))
        st = C.c_int64()
        _check(lib().dsg_model_adam_state(self.ctx.h, self.h, _p(m), _p(v), C.byref(st)))
        return m[:n], v[:n], st.value


class DeviceViews:
    """Train views resident on the device (dsg_views)."""

    def __init__(self, ctx: Context, handle: C.c_void_p, cams, width, height):
        self.ctx = ctx
        self.h = handle
        self.cams = cams
        self.width = width
        self.height = height

    @classmethod
    def from_views(cls, ctx: Context, views):
        n = len(views)
        h = C.c_void_p()
        if n == 0:
            _check(lib().dsg_views_create(ctx.h, None, None, None, C.c_int32(0), C.byref(h)))
            return cls(ctx, h, [], 0, 0)
        for v in views:
            v.validate()
        cams = (dsg_camera * n)(*[cam_struct(v.cam) for v in views])
        gts = np.ascontiguousarray(np.stack([v.ground_truth for v in views]), dtype=np.float64)
        masks = np.ascontiguousarray(np.stack([v.mask for v in views]), dtype=np.float64)
        _check(lib().dsg_views_create(ctx.h, cams, _p(gts), _p(masks), C.c_int32(n), C.byref(h)))
        return cls(ctx, h, [v.cam for v in views], views[0].cam.width, views[0].cam.height)

    @classmethod
    def synthesize(cls, ctx: Context, gt_model: "DeviceModel", cfg: RenderConfig, cams, points,
                   use_masks=True, footprint_px=2.0, dilation_px=2.0):
        """make_train_view (runtime.hpp:190-199) for every camera, on device."""
        n = len(cams)
        carr = (dsg_camera * max(n, 1))(*[cam_struct(c) for c in cams])
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        h = C.c_void_p()
        _check(lib().dsg_views_synthesize(ctx.h, gt_model.h, C.byref(cfg_struct(cfg)), carr,
                                          C.c_int32(n), _p(pts), C.c_int64(pts.shape[0]),
                                          C.c_int32(1 if use_masks else 0), C.c_double(footprint_px),
                                          C.c_double(dilation_px), C.byref(h)))
        return cls(ctx, h, list(cams), cams[0].width if n else 0, cams[0].height if n else 0)

    def download_planar(self, i: int, pin: bool = False):
        """View i in the device layout: ((3, h, w) float32, (h, w) uint8)."""
        gt = np.empty((3, self.height, self.width), np.float32)
        m = np.empty((self.height, self.width), np.uint8)
        if pin:
            gt, m = pinned(gt), pinned(m)
        _check(lib().dsg_views_download_planar(self.ctx.h, self.h, C.c_int32(i),
                                               gt.ctypes.data_as(C.c_void_p),
                                               m.ctypes.data_as(C.c_void_p)))
        return gt, m

    def download(self, i: int) -> TrainView:
        gt = np.zeros((self.height, self.width, 3))
        m = np.zeros((self.height, self.width))
        _check(lib().dsg_views_download(self.ctx.h, self.h, C.c_int32(i), _p(gt), _p(m)))
        return TrainView(self.cams[i], gt, m)

    def __len__(self):
        return len(self.cams)

    def __del__(self):
        try:
            if self.h:
                lib().dsg_views_destroy(self.h)
        except Exception:
            pass


_default_ctx = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def _as_device_model(model, ctx: Context) -> DeviceModel:
    if isinstance(model, DeviceModel):
        return model
    return DeviceModel(ctx, model)


# ---- reference-shaped API -----------------------------------------------------
def render(model, cam: Camera, cfg: RenderConfig, ctx: Context = None) -> RenderOutput:
    """render (render.hpp:160-205) on the device."""
    ctx = ctx or default_context()
    dm = _as_device_model(model, ctx)
    n, _, _ = dm.info()
    h, w = cam.height, cam.width
    rgb = np.zeros((max(h, 1), max(w, 1), 3))
    alpha = np.zeros((max(h, 1), max(w, 1)))
    nc = np.zeros((max(h, 1), max(w, 1)), np.int32)
    order = np.zeros(max(n, 1), np.int32)
    no, it = C.c_int64(), C.c_int64()
    _check(lib().dsg_render(ctx.h, dm.h, C.byref(cam_struct(cam)), C.byref(cfg_struct(cfg)),
                            _p(rgb), _p(alpha), _p(nc, C.c_int32), _p(order, C.c_int32),
                            C.byref(no), C.byref(it)))
    return RenderOutput(rgb, alpha, nc, order[: no.value].copy(), it.value)


def bin_splats(model, cam: Camera, cfg: RenderConfig, ctx: Context = None, capacity=1 << 22):
    """Per-tile compositing lists (bin_splats, render.hpp:117-135) at 16 px tiles."""
    ctx = ctx or default_context()
    dm = _as_device_model(model, ctx)
    tx = (cam.width + 15) // 16
    ty = (cam.height + 15) // 16
    counts = np.zeros(tx * ty, np.int32)
    entries = np.zeros(capacity, np.int32)
    ne = C.c_int64()
    _check(lib().dsg_bin(ctx.h, dm.h, C.byref(cam_struct(cam)), C.byref(cfg_struct(cfg)),
                         _p(counts, C.c_int32), _p(entries, C.c_int32), C.c_int64(capacity),
                         C.byref(ne)))
    return counts, entries[: ne.value].copy()


def render_mask(points, cam: Camera, footprint_px: float, dilation_px: float,
                ctx: Context = None):
    """render_mask (render.hpp:210-233) on the device."""
    ctx = ctx or default_context()
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    mask = np.zeros((max(cam.height, 1), max(cam.width, 1)))
    _check(lib().dsg_render_mask(ctx.h, _p(pts), C.c_int64(pts.shape[0]), C.byref(cam_struct(cam)),
                                 C.c_double(footprint_px), C.c_double(dilation_px), _p(mask)))
    return mask


def masked_loss(rendered, view: TrainView, loss_lambda: float, ctx: Context = None) -> LossResult:
    """masked_loss (loss.hpp:39-73) on the device."""
    ctx = ctx or default_context()
    view.validate()
    r = np.ascontiguousarray(rendered, dtype=np.float64)
    if r.shape != view.ground_truth.shape:
        raise DsplatError(ErrorCode.DimensionMismatch, "image dimensions differ")
    gt = np.ascontiguousarray(view.ground_truth, dtype=np.float64)
    m = np.ascontiguousarray(view.mask, dtype=np.float64)
    h, w = r.shape[:2]
    dL = np.zeros_like(r)
    loss = C.c_double()
    _check(lib().dsg_masked_loss(ctx.h, _p(r), _p(gt), _p(m), C.c_int32(w), C.c_int32(h),
                                 C.c_double(loss_lambda), C.byref(loss), _p(dL)))
    return LossResult(loss.value, dL)


def backward(model, cam: Camera, cfg: RenderConfig, output: RenderOutput, dL_dpixels,
             shards: int = 1, ctx: Context = None) -> GradientBuffer:
    """backward (backward.hpp:184-332) on the device."""
    ctx = ctx or default_context()
    dm = _as_device_model(model, ctx)
    n, _, _ = dm.info()
    d = np.ascontiguousarray(dL_dpixels, dtype=np.float64)
    if d.shape != (cam.height, cam.width, 3):
        raise DsplatError(ErrorCode.DimensionMismatch, "dL_dpixels must be RGB at camera resolution")
    G = np.zeros((max(n, 1), PARAMS))
    dmn = np.zeros((max(n, 1), 2))
    tc = np.zeros(max(n, 1), np.int32)
    _check(lib().dsg_backward(ctx.h, dm.h, C.byref(cam_struct(cam)), C.byref(cfg_struct(cfg)),
                              C.c_int64(output.model_iteration), _p(d), C.c_int32(shards), _p(G),
                              _p(dmn), _p(tc, C.c_int32)))
    return GradientBuffer(G[:n], dmn[:n], tc[:n])


class AdamState:
    """AdamState (adam.hpp:19-119) whose moments live with a DeviceModel."""

    kScalars = PARAMS

    def __init__(self, model: DeviceModel):
        self.model = model

    def step(self, grads: GradientBuffer, lr: GroupRates, cfg: AdamConfig = None):
        cfg = cfg or AdamConfig()
        G = np.ascontiguousarray(grads.grads, dtype=np.float64)
        r = dsg_group_rates(*lr.as_tuple())
        a = dsg_adam_config(cfg.beta1, cfg.beta2, cfg.epsilon)
        _check(lib().dsg_adam_step(self.model.ctx.h, self.model.h, _p(G), C.byref(r), C.byref(a)))

    def step_count(self) -> int:
        return self.model.info()[2]


class AdamSnapshot:
    """The optimizer state a CheckpointSink receives (trainer.hpp:119-120):
    moments and step of the device AdamState; serialize() is the reference's
    payload [step, size, m..., v...] (adam.hpp:103-112)."""

    def __init__(self, m, v, step: int):
        self.m, self.v, self.step = m, v, int(step)

    def size(self) -> int:
        return self.m.shape[0]

    def step_count(self) -> int:
        return self.step

    def serialize(self) -> np.ndarray:
        return np.concatenate([[float(self.step), float(self.size())], self.m.ravel(),
                               self.v.ravel()])


def train_device(dmodel: DeviceModel, dviews: DeviceViews, cfg: TrainConfig, shards: int = 1,
                 progress=None, loss_trace: bool = False, checkpoint=None, origin=None):
    """The device-resident training loop (dsg_train); returns (final_loss, trace).

    checkpoint(model: SplatModel, adam: AdamSnapshot, iteration, loss) is the
    reference's CheckpointSink (every checkpoint_interval steps and at the end)."""
    fl = C.c_double()
    trace = np.zeros(max(cfg.iterations, 1)) if loss_trace else None
    cb = PROGRESS_FN(lambda it, loss, user: progress(it, loss)) if progress else None

    def _ck(it, loss, model_h, user):
        snap = dmodel.download()
        snap.origin_partition = origin
        m, v, st = dmodel.adam_state()
        checkpoint(snap, AdamSnapshot(m, v, st), it, loss)

    ck = CHECKPOINT_FN(_ck) if checkpoint else None
    _check(lib().dsg_train_checkpointed(dmodel.ctx.h, dmodel.h, dviews.h,
                                        C.byref(train_struct(cfg)), C.c_int32(shards), cb, None,
                                        ck, None, C.byref(fl), _p(trace)))
    return fl.value, (trace[: cfg.iterations] if trace is not None else None)


def train_partition_full(model: SplatModel, views, cfg: TrainConfig, shards: int = 1,
                         checkpoint=None, progress=None, ctx: Context = None,
                         loss_trace: bool = False) -> TrainResult:
    """train_partition_full (trainer.hpp:140-211): host in, host out."""
    import time
    t_in = time.perf_counter()
    ctx = ctx or default_context()
    cfg.validate()
    if len(views) == 0:
        raise DsplatError(ErrorCode.NoViews, "training requires at least one view")
    if shards < 1:
        raise DsplatError(ErrorCode.InvalidArgument, "shards must be >= 1")
    t0 = time.perf_counter()
    dm = ctx.scratch_model(model)
    t1 = time.perf_counter()
    dv = HostRefViews(ctx, views)  # scheduled views streamed from host memory
    t2 = time.perf_counter()
    fl, trace = train_device(dm, dv, cfg, shards, progress, loss_trace, checkpoint=checkpoint,
                             origin=model.origin_partition)
    t3 = time.perf_counter()
    del dv  # frees the two device view slots
    t3b = time.perf_counter()
    out = dm.download()
    out.origin_partition = model.origin_partition
    res = TrainResult(out, fl, len(model), len(out))
    if trace is not None:
        res.loss_trace = trace
    t4 = time.perf_counter()
    res.model.params  # noqa: B018
    ctx.last_phases = {"enter_s": t0 - t_in, "upload_s": t1 - t0, "views_s": t2 - t1,
                       "train_s": t3 - t2, "views_free_s": t3b - t3, "download_s": t4 - t3b,
                       "result_s": time.perf_counter() - t4}
    return res


def train_partition(model: SplatModel, views, cfg: TrainConfig, shards: int = 1,
                    ctx: Context = None) -> SplatModel:
    """train_partition (trainer.hpp:214-217)."""
    return train_partition_full(model, views, cfg, shards, ctx=ctx).model


# ---- seeding (seed.hpp) ---------------------------------------------------------
def knn_mean_distances(points, k: int, ctx: Context = None):
    """knn_mean_distances (seed.hpp:16-35): exact grid k-NN on the device."""
    ctx = ctx or default_context()
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(max(pts.shape[0], 1))
    _check(lib().dsg_knn_mean(ctx.h, _p(pts), C.c_int64(pts.shape[0]), C.c_int32(k), _p(out)))
    return out[: pts.shape[0]]


def median_nn_spacing(points, ctx: Context = None) -> float:
    """median_nn_spacing (seed.hpp:39-45)."""
    ctx = ctx or default_context()
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    out = C.c_double()
    _check(lib().dsg_median_nn_spacing(ctx.h, _p(pts), C.c_int64(pts.shape[0]), C.byref(out)))
    return out.value


def seed_gaussians(points, colors, k: int = 3, ctx: Context = None, fixed_scale=None) -> DeviceModel:
    """seed_gaussians(pc, Knn, k) / (Fixed, fixed_scale) into a device model (seed.hpp:49-74)."""
    ctx = ctx or default_context()
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    col = np.ascontiguousarray(colors, dtype=np.float64).reshape(-1, 3)
    dm = DeviceModel(ctx)
    rule = 1 if fixed_scale is not None else 0
    _check(lib().dsg_seed_gaussians(ctx.h, _p(pts), _p(col), C.c_int64(pts.shape[0]),
                                    C.c_int32(rule), C.c_int32(k),
                                    C.c_double(fixed_scale or 0.01), dm.h))
    return dm


def ground_truth_model(points, colors, scale: float, opacity: float = 0.97,
                       ctx: Context = None) -> DeviceModel:
    """ground_truth_model (seed.hpp:78-94) into a device model."""
    ctx = ctx or default_context()
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    col = np.ascontiguousarray(colors, dtype=np.float64).reshape(-1, 3)
    dm = DeviceModel(ctx)
    _check(lib().dsg_ground_truth_model(ctx.h, _p(pts), _p(col), C.c_int64(pts.shape[0]),
                                        C.c_double(scale), C.c_double(opacity), dm.h))
    return dm


def view_order(seed: int, n_views: int, iterations: int):
    """View index per step (trainer.hpp:157-163, 174)."""
    out = np.zeros(max(iterations, 1), np.int32)
    _check(lib().dsg_view_order(C.c_uint64(seed), C.c_int32(n_views), C.c_int64(iterations),
                                _p(out, C.c_int32)))
    return out[:iterations]


class HostViews(DeviceViews):
    """Views kept in pinned host memory and streamed per step (end-to-end path).

    ``gts[v]`` is a (3, h, w) float32 planar array and ``masks[v]`` an (h, w)
    uint8 array (either may be None for views the schedule never touches);
    both must stay alive (and ideally be pinned) while the object lives.
    """

    def __init__(self, ctx: Context, cams, gts, masks):
        n = len(cams)
        carr = (dsg_camera * n)(*[cam_struct(c) for c in cams])
        gp = (C.c_void_p * n)(*[None if g is None else g.ctypes.data for g in gts])
        mp = (C.c_void_p * n)(*[None if m is None else m.ctypes.data for m in masks])
        h = C.c_void_p()
        _check(lib().dsg_views_create_host(ctx.h, carr, gp, mp, C.c_int32(n), C.byref(h)))
        self._keep = (gts, masks)
        super().__init__(ctx, h, list(cams), cams[0].width, cams[0].height)


class HostRefViews(DeviceViews):
    """Views in the reference's TrainView layout (loss.hpp:14-26) left in host
    memory — ground truth (h, w, 3) float64, mask (h, w) float64 — streamed by
    dsg_train one scheduled view per step (dsg_views_create_host_ref): the host
    worker pool converts the next view into a pinned slot while the current
    step runs. Views the schedule never touches are never read."""

    def __init__(self, ctx: Context, views):
        n = len(views)
        if n == 0:
            raise DsplatError(ErrorCode.NoViews, "training requires at least one view")
        for v in views:
            v.validate()
        keep = [(np.ascontiguousarray(v.ground_truth, dtype=np.float64),
                 np.ascontiguousarray(v.mask, dtype=np.float64)) for v in views]
        carr = (dsg_camera * n)(*[cam_struct(v.cam) for v in views])
        gp = (C.c_void_p * n)(*[g.ctypes.data for g, _ in keep])
        mp = (C.c_void_p * n)(*[m.ctypes.data for _, m in keep])
        h = C.c_void_p()
        _check(lib().dsg_views_create_host_ref(ctx.h, carr, gp, mp, C.c_int32(n), C.byref(h)))
        self._keep = keep
        super().__init__(ctx, h, [v.cam for v in views], views[0].cam.width, views[0].cam.height)


def launch_count() -> int:
    L = lib()
    L.dsg_launch_count.restype = C.c_int64
    return int(L.dsg_launch_count())


def set_exact_masks(enable: bool):
    """Sub-tile masks from exact row coverage (default) or the rect only."""
    _check(lib().dsg_set_exact_masks(C.c_int32(1 if enable else 0)))


class nvtx_range:
    """NVTX range (context manager) through libdsg, for ncu --nvtx filtering."""

    def __init__(self, name: str):
        self.name = name.encode()

    def __enter__(self):
        lib().dsg_nvtx_push(C.c_char_p(self.name))
        return self

    def __exit__(self, *exc):
        lib().dsg_nvtx_pop()
        return False


def frame_stats(ctx: Context):
    nv, nd = C.c_int64(), C.c_int64()
    _check(lib().dsg_frame_stats(ctx.h, C.byref(nv), C.byref(nd)))
    return {"n_visible": nv.value, "n_dup": nd.value}


def frame_work(ctx: Context):
    """(composited pairs C, termination fix-ups) of the last forward on ctx."""
    c, f, ch = C.c_int64(), C.c_int64(), C.c_int64()
    _check(lib().dsg_frame_work(ctx.h, C.byref(c), C.byref(f), C.byref(ch)))
    return {"composited": c.value, "term_fixups": f.value, "term_changed": ch.value}


def render_timed(dmodel: DeviceModel, cams, cfg: RenderConfig, repeats: int = 1) -> float:
    """Device ms to forward-render `cams` `repeats` times (render Mpix/s)."""
    n = len(cams)
    carr = (dsg_camera * n)(*[cam_struct(c) for c in cams])
    ms = C.c_double()
    _check(lib().dsg_render_timed(dmodel.ctx.h, dmodel.h, carr, C.c_int32(n),
                                  C.byref(cfg_struct(cfg)), C.c_int32(repeats), C.byref(ms)))
    return ms.value


def pinned(a: np.ndarray) -> np.ndarray:
    """Page-lock a numpy array in place; the registration is dropped when the
    array is freed (a stale registration would make later copies into the
    same address range fail)."""
    import weakref
    a = np.ascontiguousarray(a)
    ptr = a.ctypes.data
    _check(lib().dsg_host_register(C.c_void_p(ptr), C.c_int64(a.nbytes)))
    weakref.finalize(a, lib().dsg_host_unregister, C.c_void_p(ptr))
    return a


# ---- partition / merge / multi-GPU ---------------------------------------------
def partition_cloud(positions, n: int, ghost_margin: float, ctx: Context = None):
    """partition_cloud (partition.hpp:42-104) on the device (fp64, exact)."""
    from .types import Partition
    ctx = ctx or default_context()
    pts = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    npts = pts.shape[0]
    k = max(n, 1)
    ax = C.c_int32()
    lo, hi, box = np.zeros(k), np.zeros(k), np.zeros((k, 6))
    oc, gc = np.zeros(k, np.int64), np.zeros(k, np.int64)
    cap = npts
    if n > 1:  # ghost lists can exceed npts in total: size query first
        _check(lib().dsg_partition(ctx.h, _p(pts), C.c_int64(npts), C.c_int32(n),
                                   C.c_double(ghost_margin), C.byref(ax), _p(lo), _p(hi), _p(box),
                                   _p(oc, C.c_int64), _p(gc, C.c_int64), None, None, C.c_int64(0)))
        cap = max(npts, int(gc.sum()))
    cap = max(cap, 1)
    oi, gi = np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
    _check(lib().dsg_partition(ctx.h, _p(pts), C.c_int64(npts), C.c_int32(n),
                               C.c_double(ghost_margin), C.byref(ax), _p(lo), _p(hi), _p(box),
                               _p(oc, C.c_int64), _p(gc, C.c_int64), _p(oi, C.c_uint32),
                               _p(gi, C.c_uint32), C.c_int64(cap)))
    parts, o, g = [], 0, 0
    for j in range(n):
        parts.append(Partition(j, ax.value, float(lo[j]), float(hi[j]), box[j].reshape(2, 3).copy(),
                               ghost_margin, oi[o:o + oc[j]].copy(), gi[g:g + gc[j]].copy()))
        o += oc[j]
        g += gc[j]
    return parts


def merge_models(models, partitions, ctx: Context = None, out: DeviceModel = None) -> DeviceModel:
    """merge_models (partition.hpp:109-126) over device models, one process.
    `out` (optional) is reused: its buffers are kept when large enough."""
    ctx = ctx or default_context()
    if len(models) != len(partitions):
        raise DsplatError(ErrorCode.MismatchedCounts, "one model per partition required")
    dms = [m if isinstance(m, DeviceModel) else DeviceModel(ctx, m) for m in models]
    arr = (C.c_void_p * len(dms))(*[d.h.value for d in dms])
    lo = np.array([p.cut_lo for p in partitions])
    hi = np.array([p.cut_hi for p in partitions])
    out = out if out is not None else DeviceModel(ctx)
    _check(lib().dsg_merge_models(ctx.h, arr, C.c_int32(len(dms)),
                                  C.c_int32(partitions[0].cut_axis), _p(lo), _p(hi), out.h))
    return out


class Comm:
    """NCCL communicator (dsg_comm); the unique id travels over any side channel."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().dsg_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, ctx: Context, uid: bytes, nranks: int, rank: int):
        self.ctx = ctx
        self.h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().dsg_comm_create(ctx.h, buf, C.c_int32(nranks), C.c_int32(rank),
                                     C.byref(self.h)))
        self.nranks, self.rank = nranks, rank

    def close(self):
        if self.h:
            lib().dsg_comm_destroy(self.h)
            self.h = C.c_void_p()


def merge_allgather(comm: Comm, local: DeviceModel, partition) -> tuple:
    """Ghost-trim this rank's partition and all-gather the merged model."""
    merged = DeviceModel(comm.ctx)
    n, ms = C.c_int64(), C.c_double()
    _check(lib().dsg_merge_allgather(comm.ctx.h, comm.h, local.h, C.c_int32(partition.cut_axis),
                                     C.c_double(partition.cut_lo), C.c_double(partition.cut_hi),
                                     merged.h, C.byref(n), C.byref(ms)))
    return merged, n.value, ms.value


def merge_allgather_multi(comm: Comm, locals_, partitions, out: DeviceModel = None) -> tuple:
    """Several partitions per rank: locals_[j] is partition j * nranks + rank
    (partition k on GPU k mod N); merged model in partition order. `out`
    (optional) is reused: its buffers are kept when large enough."""
    merged = out if out is not None else DeviceModel(comm.ctx)
    n, ms = C.c_int64(), C.c_double()
    arr = (C.c_void_p * len(locals_))(*[m.h.value if hasattr(m.h, "value") else m.h
                                        for m in locals_])
    lo = np.array([p.cut_lo for p in partitions], np.float64)
    hi = np.array([p.cut_hi for p in partitions], np.float64)
    _check(lib().dsg_merge_allgather_multi(comm.ctx.h, comm.h, arr, C.c_int32(len(locals_)),
                                           C.c_int32(partitions[0].cut_axis), _p(lo), _p(hi),
                                           merged.h, C.byref(n), C.byref(ms)))
    return merged, n.value, ms.value


def bench_allgather(comm: Comm, nbytes: int, reps: int = 3) -> float:
    """Diagnostic: mean device ms of an all-gather of `nbytes` per rank on the
    exchange communicator (dsg_comm_bench_allgather). Collective."""
    ms = C.c_double()
    _check(lib().dsg_comm_bench_allgather(comm.ctx.h, comm.h, C.c_int64(nbytes), C.c_int32(reps),
                                          C.byref(ms)))
    return ms.value


def merge_exchange() -> str:
    """'peer' (NVLink pulls through CUDA IPC) or 'nccl' for the last merge."""
    L = lib()
    L.dsg_merge_exchange.restype = C.c_char_p
    return L.dsg_merge_exchange().decode()


def render_distributed(comm, model: DeviceModel, cam: Camera, cfg: RenderConfig, want_image=True):
    """Tile-parallel render with the bands gathered to rank 0 (comm may be None)."""
    ctx = model.ctx
    rgb = np.zeros((cam.height, cam.width, 3)) if want_image else None
    ms = C.c_double()
    _check(lib().dsg_render_distributed(ctx.h, comm.h if comm else None, model.h,
                                        C.byref(cam_struct(cam)), C.byref(cfg_struct(cfg)),
                                        _p(rgb), C.byref(ms)))
    return rgb, ms.value


# ---- I/O and evaluation (ply_io.hpp, metrics.hpp) --------------------------------
def write_splat_ply(path: str, model, ctx: Context = None):
    """write_splat_ply (ply_io.hpp:89-119) of a host or device model."""
    ctx = ctx or default_context()
    _as_device_model(model, ctx).save_ply(path)


def read_splat_ply(path: str, ctx: Context = None) -> SplatModel:
    """read_splat_ply (ply_io.hpp:121-158)."""
    ctx = ctx or default_context()
    dm = DeviceModel(ctx)
    dm.load_ply(path)
    return dm.download()


def write_cloud_ply(path: str, positions, normals=None, colors=None):
    """write_cloud_ply (ply_io.hpp:170-191)."""
    pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    nrm = None if normals is None else np.ascontiguousarray(normals, dtype=np.float64).reshape(-1, 3)
    col = None if colors is None else np.ascontiguousarray(colors, dtype=np.float64).reshape(-1, 3)
    _check(lib().dsg_cloud_save_ply(os.fsencode(path), _p(pos), None if nrm is None else _p(nrm),
                                    None if col is None else _p(col), C.c_int64(pos.shape[0])))


def read_cloud_ply(path: str):
    """read_cloud_ply (ply_io.hpp:193-221): (positions, normals, colors)."""
    n = C.c_int64()
    _check(lib().dsg_cloud_load_ply(os.fsencode(path), None, None, None, C.c_int64(0), C.byref(n)))
    out = [np.zeros((n.value, 3)) for _ in range(3)]
    _check(lib().dsg_cloud_load_ply(os.fsencode(path), *[_p(a) for a in out], C.c_int64(n.value),
                                    C.byref(n)))
    return tuple(out)


def image_metrics(a, b, ctx: Context = None):
    """(psnr, ssim) of two (h, w, 3) images (metrics.hpp:20-38) on the device."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape != b.shape or a.ndim != 3 or a.shape[2] != 3:
        raise DsplatError(ErrorCode.DimensionMismatch, "image shapes differ")
    ps, ss = C.c_double(), C.c_double()
    _check(lib().dsg_image_metrics(ctx.h, _p(a), _p(b), C.c_int32(a.shape[1]),
                                   C.c_int32(a.shape[0]), C.byref(ps), C.byref(ss)))
    return ps.value, ss.value


def eval_view(model, truth, cam: Camera, cfg: RenderConfig, ctx: Context = None):
    """(psnr, ssim) of render(model) vs render(truth) (runtime.hpp:483-492)."""
    ctx = ctx or default_context()
    dm, dt = _as_device_model(model, ctx), _as_device_model(truth, ctx)
    ps, ss = C.c_double(), C.c_double()
    _check(lib().dsg_eval_view(ctx.h, dm.h, dt.h, C.byref(cam_struct(cam)),
                               C.byref(cfg_struct(cfg)), C.byref(ps), C.byref(ss)))
    return ps.value, ss.value


def heightfield_cloud(kind: str, n: int, seed: int = 1, ctx: Context = None):
    """RT/RM-shaped cloud (positions, colors, normals) generated on the device
    (dsg_heightfield_cloud); scenes._heightfield is its numpy restatement."""
    from .scenes import HEIGHTFIELDS, heightfield_modes
    ctx = ctx or default_context()
    hp = HEIGHTFIELDS[kind]
    modes = np.ascontiguousarray(heightfield_modes(seed, hp["modes"], hp["amp"], hp["span"]))
    out = [np.empty((n, 3)) for _ in range(3)]
    _check(lib().dsg_heightfield_cloud(ctx.h, C.c_int64(n), C.c_uint64(seed), C.c_double(hp["span"]),
                                       C.c_double(hp["amp"]), C.c_double(hp["spikes"]),
                                       C.c_int32(hp["modes"]), _p(modes), *[_p(a) for a in out]))
    return out[0], out[1], out[2]
