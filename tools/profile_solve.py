"""One warm-up + one measured C2 solve (for ncu launch lists / captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, SEED  # noqa: E402
from paper_1411_0519_b200 import stmg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = CONFIGS[name]
h = stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"], cfg["t_final"])
f = h.vector(0)
h.fill_uniform(f, SEED, 0)
if cfg["random_u0"]:
    L0 = h.levels[0]
    u0 = stmg.BlockVector(h, L0["n_x"], (L0["n_x"],))
    h.fill_uniform(u0, SEED, 1)
    h.fold_u0(f, u0)
cc = stmg.CycleConfig(nu1=1, nu2=1, block_solver=os.environ.get("STMG_BLOCK", "exact"))
# host-driven cycle graphs (profiling mode): ncu sees every kernel; the
# device-side while loop body is not expanded by ncu
h.profile(os.environ.get("STMG_HOSTLOOP", "1") == "1")
for k in range(2):
    u = h.vector(0)
    rep = h.solve(f, u, cc, 1e-8)
    print(name, "solve", k, "iterations", rep.iterations, "device_ms", 1e3 * rep.device_time_seconds,
          "launches", h.launch_count(), flush=True)
