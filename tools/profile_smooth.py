"""One reference-API damped block-Jacobi sweep (stmg_block_jacobi_step, exact
blocks) on a BASELINE config, after one warm-up sweep (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, SEED  # noqa: E402
from paper_1411_0519_b200 import stmg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = CONFIGS[name]
h = stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"], cfg["t_final"])
f, u = h.vector(0), h.vector(0)
h.fill_uniform(f, SEED, 0)
h.fill_uniform(u, SEED + 1, 0)
for _ in range(2):
    h.block_jacobi_step(0, u, f, 0.5, 1)
h.synchronize()
print(name, "smooth ok", h.norm(0, u))
