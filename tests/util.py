"""Shared fixtures, restated from the reference's tests/test_util.hpp.

* ``Rng``                 — splitmix64 stream of rng.hpp:8-64 (pure Python)
* ``smooth_config``       — test_util.hpp:19-26
* ``test_camera``         — test_util.hpp:28-39
* ``random_scene``        — test_util.hpp:47-62
* ``fd_scene``            — test_util.hpp:71-86
* ``offset_ground_truth`` — test_util.hpp:91-104 (takes a render callable)
* ``full_mask`` / ``disc_mask`` — test_util.hpp:106-117
plus ``fp32_exact`` (round params through float32 so the fp32 device store
and the fp64 checker see identical values).
"""
from __future__ import annotations

import math

import numpy as np

from paper_2509_12138_b200.types import Camera, RenderConfig, SplatModel

M64 = (1 << 64) - 1


def _mix(state):
    state = (state + 0x9E3779B97F4A7C15) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


def hash_combine(seed: int, index: int) -> int:  # rng.hpp:17-20
    s = (seed ^ ((0x2545F4914F6CDD1D + index * 0x9E3779B97F4A7C15) & M64)) & M64
    return _mix(s)[1]


class Rng:
    def __init__(self, seed: int):
        self.s = (seed ^ 0x853C49E6748FEA9B) & M64
        self.s, _ = _mix(self.s)
        self.s, _ = _mix(self.s)

    def next_u64(self) -> int:
        self.s, z = _mix(self.s)
        return z

    def uniform(self, lo: float = None, hi: float = None) -> float:
        u = float(self.next_u64() >> 11) * 2.0 ** -53
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def normal(self) -> float:
        u1 = self.uniform()
        u2 = self.uniform()
        if u1 <= 0.0:
            u1 = 2.0 ** -53
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def smooth_config() -> RenderConfig:
    return RenderConfig(sigma_cutoff=6.0, alpha_cutoff=1e-12, transmittance_floor=1e-12,
                        background=(0.5, 0.5, 0.5))


def test_camera(resolution: int = 32) -> Camera:
    return Camera((0.0, 0.0, -3.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 0.9, resolution, resolution,
                  0.1, 50.0)


def _random_quat(rng: Rng):
    q = np.array([rng.normal(), rng.normal(), rng.normal(), rng.normal()])
    n = math.sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3])
    return q / n if n > 0 else np.array([1.0, 0, 0, 0])


def random_scene(seed: int, n: int = 3) -> SplatModel:
    rng = Rng(seed)
    P = np.zeros((n, 14))
    for i in range(n):
        P[i, 0] = rng.uniform(-0.5, 0.5)
        P[i, 1] = rng.uniform(-0.5, 0.5)
        P[i, 2] = rng.uniform(-0.4, 0.4)
        s = rng.uniform(0.08, 0.35)
        P[i, 3] = math.log(s * rng.uniform(0.6, 1.6))
        P[i, 4] = math.log(s * rng.uniform(0.6, 1.6))
        P[i, 5] = math.log(s * rng.uniform(0.6, 1.6))
        P[i, 6:10] = _random_quat(rng)
        P[i, 10] = rng.uniform(-1.0, 1.5)
        P[i, 11] = rng.uniform(0.2, 0.8)
        P[i, 12] = rng.uniform(0.2, 0.8)
        P[i, 13] = rng.uniform(0.2, 0.8)
    return SplatModel(P)


def fd_scene(seed: int, n: int = 3) -> SplatModel:
    rng = Rng(seed)
    P = np.zeros((n, 14))
    for i in range(n):
        P[i, 0] = rng.uniform(-0.25, 0.25)
        P[i, 1] = rng.uniform(-0.25, 0.25)
        P[i, 2] = rng.uniform(-0.3, 0.3)
        s = rng.uniform(0.3, 0.5)
        P[i, 3] = math.log(s * rng.uniform(0.85, 1.3))
        P[i, 4] = math.log(s * rng.uniform(0.85, 1.3))
        P[i, 5] = math.log(s * rng.uniform(0.85, 1.3))
        P[i, 6:10] = _random_quat(rng)
        P[i, 10] = rng.uniform(-1.0, 1.0)
        P[i, 11] = rng.uniform(0.2, 0.8)
        P[i, 12] = rng.uniform(0.2, 0.8)
        P[i, 13] = rng.uniform(0.2, 0.8)
    return SplatModel(P)


def offset_ground_truth(render_fn, model, cam: Camera, cfg: RenderConfig, seed: int):
    gt = np.array(render_fn(model, cam, cfg).color, dtype=np.float64)
    h, w = gt.shape[:2]
    for y in range(h):
        for x in range(w):
            for c in range(3):
                hv = hash_combine(seed, (y << 24) ^ (x << 8) ^ c)
                off = 0.06 if (hv & 1) else -0.06
                gt[y, x, c] = min(max(gt[y, x, c] + off, 0.0), 1.0)
    return gt


def full_mask(w: int, h: int):
    return np.ones((h, w))


def disc_mask(w: int, h: int, cx: float, cy: float, r: float):
    ys, xs = np.mgrid[0:h, 0:w]
    dx = xs + 0.5 - cx
    dy = ys + 0.5 - cy
    return ((dx * dx + dy * dy) <= r * r).astype(np.float64)


def fp32_exact(model: SplatModel) -> SplatModel:
    return SplatModel(model.params.astype(np.float32).astype(np.float64), model.iteration,
                      model.origin_partition)


def random_cloud(seed: int, n: int, lo=(-1, -1, -1), hi=(1, 1, 1)):
    """test_partition.cpp:15-23."""
    rng = Rng(seed)
    pts = np.zeros((n, 3))
    for i in range(n):
        pts[i] = [rng.uniform(lo[0], hi[0]), rng.uniform(lo[1], hi[1]), rng.uniform(lo[2], hi[2])]
    return pts
