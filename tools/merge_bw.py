"""Merge all-gather bandwidth probe (torchrun, one rank per GPU):
every rank holds `--per-rank` random splats (two partitions of half that),
merged with dsg_merge_allgather_multi; prints GB/s into each GPU per rep.
  python -m torch.distributed.run --nproc-per-node 4 tools/merge_bw.py --per-rank 26700000
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2509_12138_b200 import api  # noqa: E402
from paper_2509_12138_b200.types import Partition, SplatModel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--per-rank", type=int, default=26_700_000)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--torch-first", action="store_true")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = api.Context(local)
    uid = [api.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = api.Comm(ctx, uid[0], world, rank)
    P = 2 * world
    half = a.per_rank // 2
    locs, parts = [], []
    rng = np.random.default_rng(rank)
    for j in range(2):
        k = j * world + rank
        p = rng.random((half, 14))
        p[:, 0] = k + p[:, 0]  # slab k along x: all owned
        locs.append(api.DeviceModel(ctx, SplatModel(p, 0, k)))
        parts.append(Partition(k, 0, float(k), float(k + 1), np.zeros((2, 3)), 0.0,
                               np.zeros(0, np.uint32), np.zeros(0, np.uint32)))
    def merges():
        for r in range(a.reps):
            dist.barrier()
            merged, n, ms = api.merge_allgather_multi(comm, locs, parts)
            t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if rank == 0:
                wire = 56.0 * n * (world - 1) / world
                print(f"rep {r}: {n:,} splats, {t.item():.2f} ms, {wire / (t.item() * 1e-3) / 1e9:.1f} GB/s "
                      f"into each GPU [{os.environ.get('NCCL_ALGO', '-')}/{os.environ.get('NCCL_PROTO', '-')}"
                      f"/ch{os.environ.get('NCCL_MIN_NCHANNELS', '-')}] via {api.merge_exchange()}",
                      flush=True)
            del merged

    def fabric():
        # the fabric's own all-gather: torch.distributed (NCCL) on a buffer of one
        # merge round's size per rank, device-timed, same GB/s definition
        nbytes = half * 56
        src = torch.empty(nbytes // 4, dtype=torch.float32, device=f"cuda:{local}")
        dst = torch.empty(world * (nbytes // 4), dtype=torch.float32, device=f"cuda:{local}")
        for written in (False, True):
            for r in range(a.reps + 1):
                dist.barrier()
                if written:  # the source just written by a kernel, as the merge's pack leaves it
                    src.fill_(float(r))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                dist.all_gather_into_tensor(dst, src)
                e1.record()
                e1.synchronize()
                t = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{local}", dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                if rank == 0 and r > 0:
                    wire = nbytes * (world - 1)
                    print(f"torch all_gather_into_tensor {nbytes / 1e6:.0f} MB/rank"
                          f"{' (source just written)' if written else ''}: {t.item():.2f} ms, "
                          f"{wire / (t.item() * 1e-3) / 1e9:.1f} GB/s into each GPU", flush=True)

    def raw():
        # the exchange communicator's own all-gather on plain buffers
        nbytes = half * 56
        ms = api.bench_allgather(comm, nbytes, a.reps)
        t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(f"libdsg communicator all-gather {nbytes / 1e6:.0f} MB/rank: {t.item():.2f} ms, "
                  f"{nbytes * (world - 1) / (t.item() * 1e-3) / 1e9:.1f} GB/s into each GPU", flush=True)

    for f in ((fabric, merges, raw) if a.torch_first else (merges, fabric, raw)):
        f()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
