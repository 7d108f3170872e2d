"""Physical residual (stmg_residual) throughput, algorithmic GB/s (24 B per dof),
CUDA events around 8 launches: python tools/res_bench.py C2 C4 ..."""
import os, sys, json
sys.path.insert(0, os.getcwd())
from bench import CONFIGS, SEED
from paper_1411_0519_b200 import stmg
out = {}
for name in sys.argv[1:]:
    cfg = CONFIGS[name]
    h = stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"], cfg["t_final"])
    n0 = h.size(0)
    f, u, r = h.vector(0), h.vector(0), h.vector(0)
    h.fill_uniform(f, SEED, 0); h.fill_uniform(u, SEED + 1, 0)
    h.residual(0, u, f, r); h.synchronize()
    h.profile(True); h.profile_reset()
    for _ in range(8): h.residual(0, u, f, r)
    ms, n, b = h.profile_read(3)
    out[name] = round(b / (ms / n * 1e-3) / 1e9)
    h.profile(False)
    h.close()
print(os.environ.get("STMG_LIB", "main"), out)
