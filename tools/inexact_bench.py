"""Full solves with inexact blocks (one spatial V-cycle per time-step block,
smoother.cpp:8-92) on the BASELINE configs: device ms per solve, iterations."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, SEED  # noqa: E402
from paper_1411_0519_b200 import stmg  # noqa: E402
from paper_1411_0519_b200 import _capi as A  # noqa: E402

for name in (sys.argv[1:] or ["C2"]):
    cfg = CONFIGS[name]
    h = stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"], cfg["t_final"])
    f, u = h.vector(0), h.vector(0)
    h.fill_uniform(f, SEED, 0)
    out = {"config": name, "dofs": h.size(0)}
    for bs in ("exact", "vcycle"):
        cc = stmg.CycleConfig(nu1=1, nu2=1, block_solver=bs)
        ts = []
        for k in range(4):
            A.check(A.lib().stmg_memset_zero(h._ctx, u.ptr, u.n * 8))
            rep = h.solve(f, u, cc, 1e-8)
            ts.append(rep.device_time_seconds * 1e3)
        out[bs] = {"ms_min": min(ts[1:]), "iterations": rep.iterations, "launches": h.launch_count()}
    print(json.dumps(out), flush=True)
    h.close()
