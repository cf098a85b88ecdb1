"""Debug: device partition_cloud vs the numpy restatement at RT scale."""
import sys, os, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2509_12138_b200 import api, scenes
import host_partition as hp

n = int(sys.argv[1]) if len(sys.argv) > 1 else 18_200_000
pts, _, _ = scenes.rt(n, seed=1)
ctx = api.Context(0)
margin = 3 * 0.000172193391652984
a = api.partition_cloud(pts, 8, margin, ctx=ctx)
b = hp.partition_cloud(pts, 8, margin)
ax = b[0].cut_axis
for k, (pa, pb) in enumerate(zip(a, b)):
    eo = np.array_equal(pa.owned_indices, pb.owned_indices)
    eg = np.array_equal(pa.ghost_indices, pb.ghost_indices)
    print(k, pa.cut_axis, pb.cut_axis, pa.cut_lo == pb.cut_lo, pa.cut_hi == pb.cut_hi,
          len(pa.owned_indices), len(pb.owned_indices), eo, eg, flush=True)
    if not eo:
        sa, sb = set(pa.owned_indices.tolist()), set(pb.owned_indices.tolist())
        only_a = sorted(sa - sb)[:5]
        only_b = sorted(sb - sa)[:5]
        print("  only dev", only_a, [pts[i, ax] for i in only_a])
        print("  only ref", only_b, [pts[i, ax] for i in only_b])
        d = np.nonzero(pa.owned_indices != pb.owned_indices)[0]
        print("  first diff pos", d[:3], pa.owned_indices[d[:3]], pb.owned_indices[d[:3]])
        print("  sorted dev?", bool(np.all(np.diff(pa.owned_indices.astype(np.int64)) > 0)))
