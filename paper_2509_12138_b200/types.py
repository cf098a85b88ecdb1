"""Value types of the reference's public C++ API, mirrored for the host side.

Each type keeps the reference's field names, defaults and validation
messages so that code written against `dsplat::` reads the same here:

* ``Camera``        — camera.hpp:16-70
* ``RenderConfig``  — render.hpp:20-35
* ``AdamConfig``    — adam.hpp:11-15
* ``TrainConfig``   — trainer.hpp:13-39
* ``SplatModel``    — gaussian.hpp:41-54, stored as an (n, 14) float64 array in
  the reference's flat scalar order mu(3) log_scale(3) rot wxyz(4)
  opacity_logit(1) color(3) (adam.hpp:76-98)
* ``TrainView``     — loss.hpp:14-26 (ground truth HWC RGB, mask HW)
* ``DsplatError`` / ``ErrorCode`` — error.hpp:10-69 ("<Code>: msg")
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

PARAMS = 14  # scalars per Gaussian (AdamState::kScalars, adam.hpp:23)


class ErrorCode(enum.IntEnum):
    """dsplat::ErrorCode (error.hpp:10-31); the C ABI returns value + 1."""

    BehindCamera = 0
    InvalidRig = 1
    UnknownKind = 2
    IsovalueOutOfRange = 3
    EmptyCloud = 4
    DimensionMismatch = 5
    TooSmall = 6
    EmptyBand = 7
    EmptyInterior = 8
    MismatchedCounts = 9
    NoViews = 10
    StaleForward = 11
    IoError = 12
    MalformedFile = 13
    WorkerFailure = 14
    Timeout = 15
    ManifestMismatch = 16
    MissingBaseline = 17
    InvalidArgument = 18


class DsplatError(RuntimeError):
    """dsplat::Error: ``str(e)`` is "<Code>: msg" (error.hpp:57-61)."""

    def __init__(self, code: ErrorCode, message: str):
        super().__init__(f"{code.name}: {message}")
        self.code = code
        self.message = message


@dataclass
class Camera:
    position: tuple = (0.0, 0.0, 0.0)
    target: tuple = (0.0, 0.0, 1.0)
    up: tuple = (0.0, 1.0, 0.0)
    fov_y: float = 0.9
    width: int = 64
    height: int = 64
    near: float = 0.01
    far: float = 100.0

    def validate(self) -> None:  # camera.hpp:26-36
        if self.width < 8 or self.height < 8:
            raise DsplatError(ErrorCode.InvalidRig, "camera resolution below 8 px")
        if not (0.0 < self.fov_y < math.pi):
            raise DsplatError(ErrorCode.InvalidRig, "fov_y outside (0, pi)")
        if not (self.near < self.far):
            raise DsplatError(ErrorCode.InvalidRig, "near must be < far")

    def focal_px(self) -> float:  # camera.hpp:56
        return 0.5 * self.height / math.tan(0.5 * self.fov_y)


@dataclass
class RenderConfig:
    tile_size: int = 16
    alpha_cutoff: float = 1.0 / 255.0
    sigma_cutoff: float = 3.0
    background: tuple = (1.0, 1.0, 1.0)
    transmittance_floor: float = 1e-4

    def validate(self) -> None:  # render.hpp:27-34
        if self.tile_size <= 0 or (self.tile_size & (self.tile_size - 1)) != 0:
            raise DsplatError(ErrorCode.InvalidArgument, "tile_size must be a positive power of two")
        if not (0.0 < self.alpha_cutoff < 1.0):
            raise DsplatError(ErrorCode.InvalidArgument, "alpha_cutoff outside (0, 1)")
        if not (1.0 <= self.sigma_cutoff <= 6.0):
            raise DsplatError(ErrorCode.InvalidArgument, "sigma_cutoff outside [1, 6]")


@dataclass
class AdamConfig:
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-15


@dataclass
class GroupRates:  # AdamState::GroupRates, adam.hpp:51-53
    mu: float
    log_scale: float
    rot: float
    opacity: float
    color: float

    def as_tuple(self):
        return (self.mu, self.log_scale, self.rot, self.opacity, self.color)


@dataclass
class TrainConfig:
    iterations: int = 2000
    lr_mu: float = 1e-3
    lr_mu_decay: float = 0.01
    lr_scale: float = 5e-3
    lr_rot: float = 1e-3
    lr_opacity: float = 5e-2
    lr_color: float = 5e-3
    loss_lambda: float = 0.2
    densify_interval: int = 100
    densify_grad_threshold: float = 2e-4
    prune_opacity: float = 5e-3
    densify_stop_fraction: float = 0.5
    split_scale_threshold: float = 0.0
    checkpoint_interval: int = 0
    seed: int = 1
    render: RenderConfig = field(default_factory=RenderConfig)
    adam: AdamConfig = field(default_factory=AdamConfig)

    def validate(self) -> None:  # trainer.hpp:31-38
        if min(self.lr_mu, self.lr_scale, self.lr_rot, self.lr_opacity, self.lr_color) <= 0:
            raise DsplatError(ErrorCode.InvalidArgument, "learning rates must be positive")
        if not (0.0 <= self.loss_lambda <= 1.0):
            raise DsplatError(ErrorCode.InvalidArgument, "loss_lambda outside [0, 1]")
        if self.iterations < 0:
            raise DsplatError(ErrorCode.InvalidArgument, "iterations must be >= 0")


class SplatModel:
    """Host copy of a splat model: ``params`` is (n, 14) float64."""

    def __init__(self, params=None, iteration: int = 0, origin_partition: Optional[int] = None):
        if params is None:
            params = np.zeros((0, PARAMS))
        self.params = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, PARAMS)
        self.iteration = int(iteration)
        self.origin_partition = origin_partition

    def __len__(self) -> int:
        return self.params.shape[0]

    def size(self) -> int:
        return len(self)

    def copy(self) -> "SplatModel":
        return SplatModel(self.params.copy(), self.iteration, self.origin_partition)

    @property
    def mu(self):
        return self.params[:, 0:3]

    @property
    def log_scale(self):
        return self.params[:, 3:6]

    @property
    def rot(self):
        return self.params[:, 6:10]

    @property
    def opacity_logit(self):
        return self.params[:, 10]

    @property
    def color(self):
        return self.params[:, 11:14]


@dataclass
class TrainView:
    cam: Camera
    ground_truth: np.ndarray  # (h, w, 3) float64
    mask: np.ndarray          # (h, w) float64 in {0, 1}

    def validate(self) -> None:  # loss.hpp:19-25
        h, w = self.cam.height, self.cam.width
        if self.ground_truth.shape != (h, w, 3):
            raise DsplatError(ErrorCode.DimensionMismatch, "ground truth does not match camera")
        if self.mask.shape != (h, w):
            raise DsplatError(ErrorCode.DimensionMismatch, "mask does not match camera")


@dataclass
class RenderOutput:  # render.hpp:37-43
    color: np.ndarray                       # (h, w, 3)
    alpha: np.ndarray                       # (h, w)
    per_pixel_contributor_count: np.ndarray  # (h, w) int32
    splat_order: np.ndarray                 # (n_visible,) int32
    model_iteration: int = 0


@dataclass
class GradientBuffer:  # gradient.hpp:12-46, grads (n, 14) in parameter order
    grads: np.ndarray
    d_mean2d: np.ndarray
    touch_count: np.ndarray

    @property
    def d_mu(self):
        return self.grads[:, 0:3]

    @property
    def d_log_scale(self):
        return self.grads[:, 3:6]

    @property
    def d_rot(self):
        return self.grads[:, 6:10]

    @property
    def d_opacity_logit(self):
        return self.grads[:, 10]

    @property
    def d_color(self):
        return self.grads[:, 11:14]


@dataclass
class LossResult:  # loss.hpp:28-31
    loss: float
    dL_dpixels: np.ndarray


@dataclass
class TrainResult:  # trainer.hpp:125-130
    model: SplatModel
    final_loss: float = 0.0
    size_before_densify: int = 0
    size_after_densify: int = 0


@dataclass
class Partition:  # partition.hpp:18-30 (point arrays as index lists)
    id: int
    cut_axis: int
    cut_lo: float
    cut_hi: float
    owned_box: np.ndarray  # (2, 3) lo, hi
    ghost_margin: float
    owned_indices: np.ndarray
    ghost_indices: np.ndarray


def owns(p: Partition, position) -> bool:
    """partition.hpp:34-37: half-open ownership along the cut axis."""
    v = float(position[p.cut_axis])
    return p.cut_lo <= v < p.cut_hi
