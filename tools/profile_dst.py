"""Forward sine-basis transform of one level-0 vector (for ncu captures of the
DST passes alone): python tools/profile_dst.py C5 [reps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, SEED  # noqa: E402
from paper_1411_0519_b200 import stmg  # noqa: E402
from paper_1411_0519_b200 import _capi as A  # noqa: E402
import ctypes as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS[name]
h = stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"], cfg["t_final"])
f, u = h.vector(0), h.vector(0)
h.fill_uniform(f, SEED, 0)
cc = stmg.CycleConfig(nu1=1, nu2=1)
h.profile(True)
for k in range(reps):
    h.profile_reset()
    rep = h.solve(f, u, cc, 1e-8, max_iter=1)
    ms, n, b = h.profile_read(2)
    print(name, "transform avg ms", ms / max(n, 1), "GB/s", b / (ms / n * 1e-3) / 1e9 if n else 0,
          flush=True)
