"""Phase timeline of stmg_solve_host_batch on C2 (STMG_BATCH_TRACE=1): H2D,
solve and D2H start/end per problem, ms from the batch start."""
import ctypes as C
import os
import sys
import time

import numpy as np

os.environ["STMG_BATCH_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0519_b200 import _capi as A, stmg  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
zero = len(sys.argv) > 2 and sys.argv[2] == "zero"  # zero initial guess: nothing uploaded for u
h = stmg.Hierarchy(1, 2, 6, 8)
n = h.size(0)
bufs = []
for _ in range(5):
    p = C.c_void_p()
    A.check(A.lib().stmg_host_alloc(h._ctx, n * 8, C.byref(p)))
    bufs.append((p, np.ctypeslib.as_array((C.c_double * n).from_address(p.value))))
f = h.vector(0)
h.fill_uniform(f, 42, 0)
A.check(A.lib().stmg_download(h._ctx, bufs[0][0].value, f.ptr, n * 8))
bufs[1][1][:] = 0.0
cfg = stmg.CycleConfig(nu1=1, nu2=1)
outs = [b[1] for b in bufs[2:]]
for rep in range(2):
    h.synchronize()
    t0 = time.perf_counter()
    reps = h.solve_host_batch([bufs[0][1]] * k, [outs[i % 3] for i in range(k)], cfg, 1e-8,
                              u0s=[None if zero else bufs[1][1]] * k)
    dt = time.perf_counter() - t0
    print(f"rep {rep}: {k} solves, {1e3 * dt / k:.3f} ms per solve, iterations "
          f"{[r.iterations for r in reps]}", file=sys.stderr, flush=True)
