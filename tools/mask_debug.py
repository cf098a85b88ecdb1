"""Debug: which splats composite at a pixel (fp64, oracle prepare) but fail
the sub-tile row-interval test (fp32 emulation)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import Oracle  # noqa: E402
from paper_2509_12138_b200 import api, scenes  # noqa: E402
from paper_2509_12138_b200.types import RenderConfig  # noqa: E402

px_x, px_y, view = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ctx = api.Context(0)
pts, cols, _ = scenes.kingsnake(4_000_000, seed=1)
rig = scenes.rig_for_cloud(pts, 28, 16, 1024)
cams = [rig[i] for i in np.linspace(0, len(rig) - 1, 3).astype(int)]
seeds = api.seed_gaussians(pts, cols, 3, ctx=ctx).download()
rc = RenderConfig()
pr = Oracle().prepare(seeds, cams[view], rc)
m, ic, op = pr["mean2d"], pr["inv_cov"], pr["opacity"]
ixx, ixy, iyy = ic[:, 0], ic[:, 1], ic[:, 2]
cx, cy = px_x + 0.5, px_y + 0.5
dx, dy = cx - m[:, 0], cy - m[:, 1]
q = ixx * dx * dx + 2 * ixy * dx * dy + iyy * dy * dy
qe = np.minimum(rc.sigma_cutoff ** 2, 2 * np.log(op / rc.alpha_cutoff))
hit = np.nonzero(q <= qe)[0]
print("splats composite-eligible at pixel:", len(hit))
f = np.float32
for k in hit:
    inv = 1.0 / ixx[k]
    r = ixy[k] * inv
    qc = qe[k] + 1e-9 * abs(qe[k]) + 1e-12
    MX, MY, R, INV = f(m[k, 0]), f(m[k, 1]), f(r), f(inv)
    MXL, MYL = f(m[k, 0] - float(MX)), f(m[k, 1] - float(MY))
    Q0, QC, PAD = f(iyy[k] - ixy[k] * r), f(qc), f(1e-5 * abs(qc) * inv)
    DY = (f(f(px_y) + f(0.5)) - MY) - MYL
    H2 = (QC - DY * DY * Q0) * INV + PAD
    C = (MX - R * DY) + MXL
    H = np.sqrt(max(H2, f(0)))
    eps = f(2e-3) + f(1e-5) * (abs(C) + H)
    lo, hi = np.ceil(C - H - eps - f(0.5)), np.floor(C + H + eps - f(0.5))
    ok = H2 >= 0 and lo <= px_x <= hi
    if not ok:
        print("FAIL idx", pr["index"][k], "q", q[k], "qe", qe[k], "H2", H2, "C", C, "H", H, "lo", lo,
              "hi", hi, "ixx", ixx[k], "ixy", ixy[k], "iyy", iyy[k], "op", op[k], "mean", m[k])
print("done")
