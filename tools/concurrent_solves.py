"""Aggregate throughput of independent C2 solves run concurrently on T contexts
(one host thread and one library stream each) against one context:
python tools/concurrent_solves.py [threads ...]."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, SEED  # noqa: E402
from paper_1411_0519_b200 import stmg  # noqa: E402
from paper_1411_0519_b200 import _capi as A  # noqa: E402

name = "C2"
cfg = CONFIGS[name]
K = 40


def make():
    h = stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"], cfg["t_final"])
    f, u = h.vector(0), h.vector(0)
    h.fill_uniform(f, SEED, 0)
    cc = stmg.CycleConfig(nu1=1, nu2=1)
    h.solve(f, u, cc, 1e-8)
    return h, f, u, cc


def work(ctx, k):
    h, f, u, cc = ctx
    for _ in range(k):
        A.check(A.lib().stmg_memset_zero(h._ctx, u.ptr, u.n * 8))
        h.solve(f, u, cc, 1e-8)
    h.synchronize()


for T in [int(a) for a in (sys.argv[1:] or ["1", "2", "3"])]:
    ctxs = [make() for _ in range(T)]
    for c in ctxs:
        work(c, 2)
    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(c, K // T)) for c in ctxs]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    print(f"{T} context(s): {K // T * T} solves in {dt * 1e3:.1f} ms = {dt * 1e3 / (K // T * T):.3f} ms per solve",
          flush=True)
    for c in ctxs:
        c[0].close()
