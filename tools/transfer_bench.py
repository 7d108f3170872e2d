"""Reference-API transfer operators (stmg_restrict / stmg_prolong, physical
space) on level 0 of the BASELINE configs: algorithmic GB/s (fine read/write
8 B per fine dof + coarse 8 B per coarse dof), wall clock around 5 launches;
and the physical-path full solve (cfg.path = physical) next to the spectral one."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, SEED  # noqa: E402
from paper_1411_0519_b200 import stmg  # noqa: E402
from paper_1411_0519_b200 import _capi as A  # noqa: E402

for name in (sys.argv[1:] or ["C2"]):
    cfg = CONFIGS[name]
    h = stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"], cfg["t_final"])
    n0 = h.size(0)
    f = h.vector(0)
    h.fill_uniform(f, SEED, 0)
    out = {"config": name, "dofs": n0, "coarsen_to_next": h.levels[0]["coarsen_to_next"]}
    mode = h.levels[0]["coarsen_to_next"]
    c = h.coarse_vector(0, mode)
    fine = h.vector(0)
    for nm, fn in (("restrict", lambda: A.check(A.lib().stmg_restrict(h._ctx, 0, mode, f.ptr, c.ptr))),
                   ("prolong", lambda: A.check(A.lib().stmg_prolong(h._ctx, 0, mode, c.ptr, fine.ptr)))):
        fn()
        h.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            fn()
        h.synchronize()
        dt = (time.perf_counter() - t0) / 5
        out[nm] = {"ms": dt * 1e3, "alg_GBps": 8.0 * (n0 + c.n) / dt / 1e9}
    del c, fine
    # semi-coarsening variants (time only), norm, forward substitution
    c1 = h.coarse_vector(0, 1)
    fine = h.vector(0)

    def timed(fn, reps=5):
        fn()
        h.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        h.synchronize()
        return (time.perf_counter() - t0) / reps

    dt = timed(lambda: A.check(A.lib().stmg_restrict(h._ctx, 0, 1, f.ptr, c1.ptr)))
    out["restrict_semi"] = {"ms": dt * 1e3, "alg_GBps": 8.0 * (n0 + c1.n) / dt / 1e9}
    dt = timed(lambda: A.check(A.lib().stmg_prolong(h._ctx, 0, 1, c1.ptr, fine.ptr)))
    out["prolong_semi"] = {"ms": dt * 1e3, "alg_GBps": 8.0 * (n0 + c1.n) / dt / 1e9}
    dt = timed(lambda: h.norm(0, f))
    out["norm"] = {"ms": dt * 1e3, "alg_GBps": 8.0 * n0 / dt / 1e9}
    last = len(h.levels) - 1
    fl = h.vector(last)
    h.fill_uniform(fl, SEED, 3)
    dt = timed(lambda: h.forward_substitution_solve(last, fl))
    out["forward_substitution_coarsest"] = {"ms": dt * 1e3, "dofs": fl.n}
    del c1, fine, fl
    if name == "C2":
        u = h.vector(0)
        for path in ("spectral", "physical"):
            cc = stmg.CycleConfig(nu1=1, nu2=1, path=path)
            ts = []
            for k in range(3):
                A.check(A.lib().stmg_memset_zero(h._ctx, u.ptr, u.n * 8))
                rep = h.solve(f, u, cc, 1e-8)
                ts.append(rep.device_time_seconds * 1e3)
            out[path] = {"ms_min": min(ts[1:]), "iterations": rep.iterations}
    print(json.dumps(out), flush=True)
    h.close()
