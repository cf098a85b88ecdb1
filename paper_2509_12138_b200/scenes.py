"""Deterministic synthetic isosurface point clouds for the BASELINE configs.

The reference builds its inputs with make_volume + marching cubes
(volume.hpp:99-145, marching_cubes.hpp:52-109), which cannot reach the 4M -
106.7M point configs (SURVEY §7 hard part 5). These generators sample the
named analytic isosurfaces directly, area-uniformly on a jittered lattice,
with analytic normals and the reference's normal-matte transfer function
(marching_cubes.hpp:26-36), so every config is reproducible from its seed:

* ``sphere``    — config 1: |p| = 0.35 (the sphere volume's default
                  isovalue, volume.hpp:83-89), Fibonacci lattice, 99,726 points
* ``kingsnake`` — config 2: a coiled tube (distance-to-helix isosurface) with
                  a banded radius, ~4M points
* ``rt``        — config 3: Rayleigh-Taylor-like mixing interface
                  y = h(x, z) with multimode bubbles/spikes, ~18.2M points
* ``rm``        — config 4: Richtmyer-Meshkov-like shocked interface with
                  finer modes, ~106.7M points
  (both also generated on the device, csrc/scene.cu: point i depends only on
  (seed, i) through the reference's hash_combine, rng.hpp:17-20)

Clouds are returned as float64 arrays (positions, colors, normals) rounded to
fp32-exact values, so the fp32 device store and the fp64 checker see the same
inputs.
"""
from __future__ import annotations

import math

import numpy as np

SIZES = {"sphere": 99_726, "kingsnake": 4_000_000, "rt": 18_200_000, "rm": 106_700_000}


def normal_matte(n: np.ndarray) -> np.ndarray:
    """transfer::normal_matte (marching_cubes.hpp:26-36), vectorised."""
    l1 = np.array([0.5, 0.7, -0.5])
    l1 /= np.linalg.norm(l1)
    l2 = np.array([-0.6, 0.2, 0.75])
    l2 /= np.linalg.norm(l2)
    lam = 0.25 + 0.55 * np.abs(n @ l1) + 0.2 * np.abs(n @ l2)
    base = 0.35 + 0.3 * (0.5 + 0.5 * n)
    return np.clip(base * lam[:, None], 0.0, 1.0)


def _finish(p, nrm):
    nrm = nrm / np.maximum(np.linalg.norm(nrm, axis=1, keepdims=True), 1e-300)
    col = normal_matte(nrm)
    f = lambda a: np.ascontiguousarray(a.astype(np.float32).astype(np.float64))
    return f(p), f(col), f(nrm)


def sphere(n: int = SIZES["sphere"], radius: float = 0.35, seed: int = 1):
    """Fibonacci lattice on the r=0.35 sphere isosurface."""
    i = np.arange(n, dtype=np.float64) + 0.5
    z = 1.0 - 2.0 * i / n
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = i * math.pi * (3.0 - math.sqrt(5.0)) + 0.1 * seed
    nrm = np.stack([r * np.cos(phi), z, r * np.sin(phi)], axis=1)
    return _finish(radius * nrm, nrm)


def _jitter(rng, shape, amp):
    return (rng.random(shape) - 0.5) * amp


def kingsnake(n: int = SIZES["kingsnake"], seed: int = 1, turns: float = 6.0):
    """Coiled tube: isosurface |p - helix(t)| = r(t), r banded like snake scales.

    Coil radius, tube radius and pitch are fixed; `turns` sets the length
    (6 turns = one unit), so a weak-scaled scene (N x points, N x turns) keeps
    the point density and per-slab geometry of the single-GPU config.
    Points are spread area-uniformly: a (t, phi) lattice whose spacing is
    matched along and around the tube, with sub-cell jitter.
    """
    rng = np.random.default_rng(seed)
    length = turns / 6.0
    R = 0.22                    # coil radius
    pitch = length / turns      # rise per turn
    r0 = 0.045                  # tube radius
    circ = 2 * math.pi * r0
    arc_per_turn = math.sqrt((2 * math.pi * R) ** 2 + pitch ** 2)
    L = arc_per_turn * turns
    ds = math.sqrt(L * circ / n)
    nt = max(8, int(round(L / ds)))
    nphi = max(8, int(math.ceil(n / nt)))
    t = (np.arange(nt)[:, None] + 0.5 + _jitter(rng, (nt, nphi), 0.5)) / nt
    ph = (np.arange(nphi)[None, :] + 0.5 + _jitter(rng, (nt, nphi), 0.5)) / nphi * 2 * math.pi
    t = t.ravel()[:n]
    ph = ph.ravel()[:n]
    th = t * turns * 2 * math.pi
    c = np.stack([R * np.cos(th), (t - 0.5) * length, R * np.sin(th)], axis=1)
    tan = np.stack([-R * np.sin(th) * turns * 2 * math.pi, np.full_like(th, length),
                    R * np.cos(th) * turns * 2 * math.pi], axis=1)
    tan /= np.linalg.norm(tan, axis=1, keepdims=True)
    nn = np.stack([np.cos(th), np.zeros_like(th), np.sin(th)], axis=1)  # inward normal of coil
    nn -= (nn * tan).sum(1, keepdims=True) * tan
    nn /= np.linalg.norm(nn, axis=1, keepdims=True)
    bn = np.cross(tan, nn)
    band = 1.0 + 0.12 * np.sin(th * 9.0) + 0.05 * np.sin(ph * 6.0 + th * 3.0)
    rad = r0 * band
    nrm = np.cos(ph)[:, None] * nn + np.sin(ph)[:, None] * bn
    p = c + rad[:, None] * nrm
    return _finish(p, nrm)


_M64 = (1 << 64) - 1


def _splitmix_np(s):
    """splitmix64 (rng.hpp:8-14) on a uint64 array (wrapping arithmetic)."""
    s = s + np.uint64(0x9E3779B97F4A7C15)
    z = s
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _hash_uniform(seed: int, index):
    """hash_combine(seed, index) (rng.hpp:17-20) as a uniform in [0, 1)."""
    with np.errstate(over="ignore"):
        s = np.uint64(seed & _M64) ^ (np.uint64(0x2545F4914F6CDD1D) + index.astype(np.uint64)
                                      * np.uint64(0x9E3779B97F4A7C15))
        return (_splitmix_np(s) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def heightfield_modes(seed: int, modes: int, amp: float, span: float):
    """Mode table [modes][5] = (kx, kz, phase_x, phase_z, amplitude), drawn
    with the reference's Rng (rng.hpp:22-64) seeded seed + 7."""
    st = [(((seed + 7) ^ 0x853C49E6748FEA9B) & _M64)]

    def nxt():
        st[0] = (st[0] + 0x9E3779B97F4A7C15) & _M64
        z = st[0]
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    nxt()
    nxt()
    uni = lambda: float(nxt() >> 11) * 2.0 ** -53  # noqa: E731
    out = np.zeros((modes, 5))
    for m in range(modes):
        kx = (1 + nxt() % 8) * (2 * math.pi / span)
        kz = (1 + nxt() % 8) * (2 * math.pi / span)
        out[m] = (kx, kz, uni() * 2 * math.pi, uni() * 2 * math.pi,
                  amp * uni() / (1.0 + 0.15 * (kx + kz)))
    return out


HEIGHTFIELDS = {"rt": dict(modes=24, amp=0.08, span=1.0, spikes=0.6),
                "rm": dict(modes=64, amp=0.06, span=1.0, spikes=0.9)}


def _heightfield(n, seed, modes, amp, span, spikes):
    """Interface y = h(x, z) on a jittered lattice; the numpy restatement of
    the device generator csrc/scene.cu (dsg_heightfield_cloud), which
    bench.py uses for the large clouds. Point i depends only on (seed, i)."""
    side = int(math.ceil(math.sqrt(n)))
    i = np.arange(n, dtype=np.int64)
    row, col = i // side, i % side
    inv = 1.0 / side
    u1 = _hash_uniform(seed, 2 * i)
    u2 = _hash_uniform(seed, 2 * i + 1)
    x = (row + 0.5) * inv + (u1 - 0.5) * 0.8 * inv
    z = (col + 0.5) * inv + (u2 - 0.5) * 0.8 * inv
    X = (x - 0.5) * span
    Z = (z - 0.5) * span
    h = np.zeros(n)
    hx = np.zeros(n)
    hz = np.zeros(n)
    for kx, kz, ph1, ph2, a in heightfield_modes(seed, modes, amp, span):
        s1, c1 = np.sin(kx * X + ph1), np.cos(kx * X + ph1)
        s2, c2 = np.sin(kz * Z + ph2), np.cos(kz * Z + ph2)
        h += a * c1 * c2
        hx += -a * kx * s1 * c2
        hz += -a * kz * c1 * s2
    # bubbles (rounded, up) and spikes (sharp, down): nonlinear RT/RM shape
    t = np.tanh(3.0 * h / amp)
    h2 = h + spikes * t * np.abs(h)
    d = 1.0 + spikes * (t * np.sign(h) + 3.0 * np.abs(h) / amp / np.cosh(3.0 * h / amp) ** 2)
    hx *= d
    hz *= d
    p = np.stack([X, h2, Z], axis=1)
    nrm = np.stack([-hx, np.ones(n), -hz], axis=1)
    return _finish(p, nrm)


def heightfield_device(kind: str, n: int, seed: int = 1, ctx=None):
    """The same cloud generated on the B200 (dsg_heightfield_cloud)."""
    from . import api
    return api.heightfield_cloud(kind, n, seed, ctx=ctx)


def rt(n: int = SIZES["rt"], seed: int = 1):
    """Rayleigh-Taylor-shaped mixing interface (multimode, bubbles and spikes)."""
    return _heightfield(n, seed, **HEIGHTFIELDS["rt"])


def rm(n: int = SIZES["rm"], seed: int = 1):
    """Richtmyer-Meshkov-shaped shocked interface (more, finer modes)."""
    return _heightfield(n, seed, **HEIGHTFIELDS["rm"])


GENERATORS = {"sphere": sphere, "kingsnake": kingsnake, "rt": rt, "rm": rm}


def make_cloud(kind: str, n: int = None, seed: int = 1, ctx=None):
    """Cloud of a named kind; with a device context the RT/RM heightfields
    are generated on the GPU (same definition, ~1e3x faster at 106.7M)."""
    if kind not in GENERATORS:
        raise ValueError(f"unknown scene kind {kind!r}")
    if ctx is not None and kind in HEIGHTFIELDS:
        return heightfield_device(kind, n or SIZES[kind], seed, ctx)
    return GENERATORS[kind](n or SIZES[kind], seed=seed)


def rig_for_cloud(positions, n_azimuth, n_elevation, resolution, fov_y=0.9, radius_scale=2.5,
                  max_elevation=math.pi / 3.0):
    """build_rig_for_cloud (runtime.hpp:65-71) + build_orbital_cameras (camera.hpp:75-107)."""
    from .types import Camera

    lo = positions.min(axis=0)
    hi = positions.max(axis=0)
    center = (lo + hi) * 0.5
    br = 0.5 * float(np.sqrt(((hi - lo) ** 2).sum()))
    if br <= 0.0:
        br = 1.0
    radius = radius_scale * br
    cams = []
    for ie in range(n_elevation):
        phi = 0.0
        if n_elevation > 1:
            phi = -max_elevation + 2.0 * max_elevation * ie / (n_elevation - 1)
        for ia in range(n_azimuth):
            th = 2.0 * math.pi * ia / n_azimuth
            d = (math.cos(phi) * math.cos(th), math.sin(phi), math.cos(phi) * math.sin(th))
            pos = tuple(float(center[k] + d[k] * radius) for k in range(3))
            cams.append(Camera(pos, tuple(float(c) for c in center), (0.0, 1.0, 0.0), fov_y,
                               resolution, resolution, 0.05 * radius, 10.0 * radius))
    return cams
