"""A/B: device-side while-loop solve graph vs per-cycle graph launches."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, SEED  # noqa: E402
from paper_1411_0519_b200 import stmg  # noqa: E402
from paper_1411_0519_b200 import _capi as A  # noqa: E402

for name in sys.argv[1:] or ["C2"]:
    cfg = CONFIGS[name]
    res = {}
    for loop in ("1", "0"):
        os.environ["STMG_DEVICE_LOOP"] = loop
        h = stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"],
                           cfg["t_final"])
        f, u = h.vector(0), h.vector(0)
        h.fill_uniform(f, SEED, 0)
        cc = stmg.CycleConfig(nu1=1, nu2=1)
        ts = []
        for k in range(8):
            A.check(A.lib().stmg_memset_zero(h._ctx, u.ptr, u.n * 8))
            rep = h.solve(f, u, cc, 1e-8)
            if k >= 3:
                ts.append(rep.device_time_seconds)
        res[loop] = (min(ts) * 1e3, sum(ts) / len(ts) * 1e3, rep.iterations)
        h.close()
    print(name, "device-loop", res["1"], "per-cycle", res["0"], flush=True)
