"""Host<->device model transfer timing (the e2e leg's upload/download)."""
import ctypes as C
import time

import numpy as np

from paper_2509_12138_b200 import api
from paper_2509_12138_b200.types import SplatModel

n = 4_000_000
ctx = api.Context(0)
P = np.random.default_rng(0).normal(size=(n, 14))
m = SplatModel(P)
dm = api.DeviceModel(ctx)
dm.upload(m)
for r in range(4):
    t0 = time.perf_counter(); dm.upload(m); t1 = time.perf_counter()
    out = dm.download(); t2 = time.perf_counter()
    Q = np.empty((n, 14)); Q[:] = 0
    nn, it, op = C.c_int64(), C.c_int64(), C.c_int32()
    t3 = time.perf_counter()
    api.lib().dsg_model_download(ctx.h, dm.h, api._p(Q), C.c_int64(n), C.byref(nn), C.byref(it), C.byref(op))
    t4 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.2f} ms  download(fresh) {1e3*(t2-t1):.2f} ms  download(prefaulted) {1e3*(t4-t3):.2f} ms")
assert np.array_equal(out.params, P.astype(np.float32).astype(np.float64))

# fresh-output cost: the page faults of a new (n, 14) float64 array
for hp in (True, False):
    np.core.multiarray._set_madvise_hugepage(hp)
    for r in range(3):
        t0 = time.perf_counter(); out = dm.download(); t1 = time.perf_counter()
        Z = np.empty((n, 14)); t2 = time.perf_counter(); Z.fill(0.0); t3 = time.perf_counter()
        print(f"hugepage={hp}: download(fresh) {1e3*(t1-t0):.2f} ms, single-thread first touch {1e3*(t3-t2):.2f} ms")
        del out, Z
