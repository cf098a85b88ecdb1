"""CPU tests of the host-side logic around the device path.

* partition.py (partition_cloud / merge_models, partition.hpp:34-126) against
  the oracle, bit-exact;
* bench.split_rig and scenes.rig_for_cloud against split_rig /
  build_orbital_cameras (camera.hpp:75-130);
* the synthetic scene generators (determinism, sizes, fp32-exactness);
* the multi-rank merge path with world_size 2 over gloo: each rank trims its
  own partition and the gathered result equals merge_models.
"""
import os
import socket

import numpy as np
import pytest

import bench
from oracle import Oracle
import host_partition as part_mod
from paper_2509_12138_b200 import scenes
from paper_2509_12138_b200.types import DsplatError, SplatModel
from util import random_cloud


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.mark.parametrize("nparts,margin", [(1, 0.25), (2, 0.0), (3, 0.15), (4, 0.2), (8, 0.3)])
def test_partition_matches_oracle(orc, nparts, margin):
    pts = random_cloud(nparts + 5, 337)
    pts[::11, 0] = pts[0, 0]
    a = part_mod.partition_cloud(pts, nparts, margin)
    b = orc.partition_cloud(pts, nparts, margin)
    for pa, pb in zip(a, b):
        assert pa.cut_axis == pb.cut_axis and pa.cut_lo == pb.cut_lo and pa.cut_hi == pb.cut_hi
        np.testing.assert_array_equal(pa.owned_box, pb.owned_box)
        np.testing.assert_array_equal(pa.owned_indices, pb.owned_indices)
        np.testing.assert_array_equal(pa.ghost_indices, pb.ghost_indices)


def test_partition_quarters_and_errors():
    # test_partition.cpp:33-44: uniform line cloud splits into exact quarters
    pts = np.array([[i * 0.001, 0.3 * ((i * 7) % 11) / 11.0, 0.0] for i in range(1000)])
    parts = part_mod.partition_cloud(pts, 4, 0.0)
    assert [len(p.owned_indices) for p in parts] == [250] * 4
    assert parts[0].cut_axis == 0
    with pytest.raises(DsplatError, match="EmptyCloud"):
        part_mod.partition_cloud(np.zeros((0, 3)), 2, 0.1)
    with pytest.raises(DsplatError, match="InvalidArgument"):
        part_mod.partition_cloud(random_cloud(1, 3), 4, 0.1)


def test_merge_matches_oracle(orc):
    pts = random_cloud(41, 200)
    parts = part_mod.partition_cloud(pts, 3, 0.2)
    rng = np.random.default_rng(1)
    models = [SplatModel(rng.uniform(-1.2, 1.2, size=(40 + 3 * k, 14)), 5 + k, k) for k in range(3)]
    merged = part_mod.merge_models(models, parts)
    keep = orc.merge_keep([m.params for m in models], parts)
    np.testing.assert_array_equal(merged.params, np.concatenate([m.params for m in models])[keep])
    assert merged.iteration == 7
    with pytest.raises(DsplatError, match="MismatchedCounts"):
        part_mod.merge_models(models[:2], parts)


def test_split_rig_and_rig_match_oracle(orc):
    for n, frac, seed in ((64, 0.1, 1), (28, 4 / 28, 11), (448, 0.1, 3), (1, 0.5, 2)):
        tr, te = bench.split_rig(n, frac, seed)
        otr, ote = orc.split_rig(n, frac, seed)
        np.testing.assert_array_equal(tr, otr)
        np.testing.assert_array_equal(te, ote)
    pts, _, _ = scenes.sphere(5000)
    cams = scenes.rig_for_cloud(pts, 7, 5, 32)
    lo, hi = pts.min(0), pts.max(0)
    center = (lo + hi) * 0.5
    radius = 2.5 * 0.5 * float(np.sqrt(((hi - lo) ** 2).sum()))
    ref = orc.build_orbital_cameras(center, radius, 7, 5, 32)
    for a, b in zip(cams, ref):
        np.testing.assert_allclose(a.position, b.position, rtol=0, atol=1e-15)
        assert a.near == b.near and a.far == b.far and a.width == b.width


@pytest.mark.parametrize("kind,n", [("sphere", 99_726), ("kingsnake", 20_000), ("rt", 20_000),
                                    ("rm", 20_000)])
def test_scenes_deterministic_and_fp32_exact(kind, n):
    a = scenes.make_cloud(kind, n, seed=3)
    b = scenes.make_cloud(kind, n, seed=3)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    pos, col, nrm = a
    assert pos.shape == (n, 3) and col.shape == (n, 3)
    np.testing.assert_array_equal(pos, pos.astype(np.float32).astype(np.float64))
    assert np.all((col >= 0) & (col <= 1))
    np.testing.assert_allclose(np.linalg.norm(nrm, axis=1), 1.0, atol=1e-6)


def test_kingsnake_weak_scaling_keeps_density():
    p1, _, _ = scenes.kingsnake(40_000, turns=6.0)
    p2, _, _ = scenes.kingsnake(80_000, turns=12.0)
    e1 = p1.max(0) - p1.min(0)
    e2 = p2.max(0) - p2.min(0)
    assert abs(e1[0] - e2[0]) < 0.02 and abs((e2[1] - e1[1]) - 1.0) < 0.02  # same coil, +1 unit


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _merge_worker(rank, world, port, pts, models, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    parts = part_mod.partition_cloud(pts, world, 0.1)       # every rank cuts the same slabs
    mine = models[rank]
    kept = mine.params[part_mod.merge_keep(mine.params, parts[rank])]
    gathered = [None] * world
    dist.all_gather_object(gathered, kept)                  # partition (= rank) order
    if rank == 0:
        out.put(np.concatenate(gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_merge_gloo_world2(orc):
    import multiprocessing as mp
    pts = random_cloud(7, 300)
    rng = np.random.default_rng(3)
    models = [SplatModel(rng.uniform(-1.1, 1.1, size=(60 + 5 * k, 14)), 3, k) for k in range(2)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_merge_worker, args=(r, 2, port, pts, models, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = orc.partition_cloud(pts, 2, 0.1)
    keep = orc.merge_keep([m.params for m in models], parts)
    np.testing.assert_array_equal(got, np.concatenate([m.params for m in models])[keep])


def test_view_order_host_matches_library():
    """bench.py's reference arm restates the seeded view order in Python so
    it never maps libdsg.so; it must equal dsg_view_order (host code, no GPU)."""
    from paper_2509_12138_b200 import api
    for seed, n, iters in ((1, 403, 50), (7, 58, 130), (2, 1, 3), (123456789, 17, 40)):
        assert bench.view_order_host(seed, n, iters) == api.view_order(seed, n, iters).tolist()


def test_reference_arm_seeds_match_seed_gaussians():
    """The reference arm's k-d-tree kNN seeds equal the reference's O(N^2)
    seed_gaussians (seed.hpp:49-74) bit for bit on a cloud it can still run."""
    from oracle import Reference, has_reference
    pts, cols, _ = scenes.kingsnake(3000, seed=2)
    impl = Reference() if has_reference() else Oracle()
    np.testing.assert_array_equal(bench.knn_seeds_host(pts, cols).params,
                                  impl.seed_gaussians(pts, cols, 3).params)
