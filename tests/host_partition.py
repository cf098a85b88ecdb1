"""TEST INFRASTRUCTURE: a numpy restatement of slab partitioning with ghost
cells and the ghost-trimming merge, used by the CPU (gloo) multi-process tests
and the multi-GPU checker. The product path is the device partitioner
(csrc/partition.cu) and dsg_merge_allgather (csrc/comm.cu).

partition_cloud (partition.hpp:42-104), owns (:34-37) and merge_models
(:109-126) with the reference's exact semantics:

* axis = longest AABB extent, ties x > y > z (math.hpp:164-170)
* points ordered by (coordinate, index); cut_k = 0.5 * (v[r-1] + v[r]) with
  r = floor(n * k / parts) — fp64, so membership is bit-identical
* ownership is half-open [cut_lo, cut_hi) with open outer slabs
* ghosts: foreign points within `ghost_margin` of the owned interval
* merge keeps a splat iff its final mu is owned by its origin partition,
  in (partition, index) order

Vectorised numpy over fp64 positions: this is one-time O(N log N) setup per
job, not part of the per-step device path.
"""
from __future__ import annotations

import numpy as np

from paper_2509_12138_b200.types import PARAMS, DsplatError, ErrorCode, Partition, SplatModel


def partition_cloud(positions, n: int, ghost_margin: float):
    pts = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    N = pts.shape[0]
    if N == 0:
        raise DsplatError(ErrorCode.EmptyCloud, "cannot partition an empty cloud")
    if n < 1:
        raise DsplatError(ErrorCode.InvalidArgument, "partition count must be >= 1")
    if n > N:
        raise DsplatError(ErrorCode.InvalidArgument, "more partitions than points")
    if ghost_margin < 0.0:
        raise DsplatError(ErrorCode.InvalidArgument, "ghost margin must be >= 0")
    lo = pts.min(axis=0)
    hi = pts.max(axis=0)
    e = hi - lo
    if e[0] >= e[1] and e[0] >= e[2]:
        axis = 0
    else:
        axis = 1 if e[1] >= e[2] else 2
    v = pts[:, axis]
    order = np.lexsort((np.arange(N), v))  # by (coordinate, index)
    cuts = []
    for k in range(1, n):
        r = (N * k) // n
        cuts.append(0.5 * (v[order[r - 1]] + v[order[r]]))
    parts = []
    for k in range(n):
        c_lo = -np.inf if k == 0 else cuts[k - 1]
        c_hi = np.inf if k == n - 1 else cuts[k]
        box = np.stack([lo.copy(), hi.copy()])
        if k > 0:
            box[0, axis] = cuts[k - 1]
        if k < n - 1:
            box[1, axis] = cuts[k]
        own = (v >= c_lo) & (v < c_hi)
        blo, bhi = box[0, axis], box[1, axis]
        dist = np.where(v < blo, blo - v, np.where(v > bhi, v - bhi, 0.0))
        ghost = (~own) & (dist <= ghost_margin)
        parts.append(Partition(k, axis, float(c_lo), float(c_hi), box, ghost_margin,
                               np.nonzero(own)[0].astype(np.uint32),
                               np.nonzero(ghost)[0].astype(np.uint32)))
    return parts


def owns(p: Partition, position) -> bool:
    v = float(position[p.cut_axis])
    return p.cut_lo <= v < p.cut_hi


def merge_keep(params: np.ndarray, p: Partition) -> np.ndarray:
    v = np.asarray(params, dtype=np.float64).reshape(-1, PARAMS)[:, p.cut_axis]
    return (v >= p.cut_lo) & (v < p.cut_hi)


def merge_models(models, partitions) -> SplatModel:
    if len(models) != len(partitions):
        raise DsplatError(ErrorCode.MismatchedCounts, "one model per partition required")
    kept = []
    it = 0
    for m, p in zip(models, partitions):
        if m.origin_partition is None:
            raise DsplatError(ErrorCode.MismatchedCounts, "model missing origin partition id")
        if m.origin_partition != p.id:
            raise DsplatError(ErrorCode.MismatchedCounts, "model/partition id mismatch")
        kept.append(m.params[merge_keep(m.params, p)])
        it = max(it, m.iteration)
    P = np.concatenate(kept) if kept else np.zeros((0, PARAMS))
    return SplatModel(P, it)
