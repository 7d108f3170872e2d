"""Per-kernel HBM throughput on the BASELINE configs (run on the GPU box).

For each config: the fused level-0 V-cycle kernel (k_updown; k_down / k_up
for the per-level schedule) and the coarse part of each cycle (levels >= 1),
timed live with CUDA events inside the cycle graph, one full sine-basis transform
(dim DST-I passes), the physical Q1 residual kernel (stmg_residual) and the
physical block-Jacobi sweep (stmg_smooth, nu = 1).  Achieved GB/s use
ALGORITHMIC bytes.  Prints one JSON line per config.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, SEED, peaks  # noqa: E402
from paper_1411_0519_b200 import stmg  # noqa: E402
from paper_1411_0519_b200 import _capi as A  # noqa: E402


def run(name, reps=5):
    cfg = CONFIGS[name]
    h = stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"], cfg["t_final"])
    n0 = h.size(0)
    f, u = h.vector(0), h.vector(0)
    h.fill_uniform(f, SEED, 0)
    cc = stmg.CycleConfig(nu1=1, nu2=1)
    h.solve(f, u, cc, 1e-8)  # warm-up (graph capture, buffers)
    h.profile(True)
    h.profile_reset()
    for _ in range(reps):
        A.check(A.lib().stmg_memset_zero(h._ctx, u.ptr, n0 * 8))
        rep = h.solve(f, u, cc, 1e-8)
    out = {"config": name, "dofs": n0, "iterations": rep.iterations,
           "solve_ms": rep.device_time_seconds * 1e3}
    fused = h.profile_read(1)[1] == 0
    names = ({0: "k_updown_l0", 2: "transform", 4: "coarse_part"} if fused else
             {0: "k_down_l0", 1: "k_up_l0", 2: "transform"})
    for k, nm in names.items():
        ms, n, b = h.profile_read(k)
        if n:
            out[nm] = {"avg_ms": ms / n, "launches": n}
            if b:
                out[nm]["alg_GBps"] = b / (ms / n * 1e-3) / 1e9
    # physical residual (24 B/dof: read u, f; write r)
    r = h.vector(0)
    h.residual(0, u, f, r)  # warm-up (lazy module load, attributes)
    h.synchronize()
    h.profile_reset()
    for _ in range(reps):
        h.residual(0, u, f, r)
    ms, n, b = h.profile_read(3)
    out["residual_phys"] = {"avg_ms": ms / n, "alg_GBps": b / (ms / n * 1e-3) / 1e9}
    del r
    # physical smoother sweep: residual + forward/inverse transforms + solve + update
    h.block_jacobi_step(0, u, f, 0.5, 1)  # warm-up
    h.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        h.block_jacobi_step(0, u, f, 0.5, 1)
    h.synchronize()
    dt = (time.perf_counter() - t0) / reps
    out["smooth_phys"] = {"avg_ms": dt * 1e3, "alg_GBps_24B": 24 * n0 / dt / 1e9}
    h.profile(False)
    peak, kind = peaks()
    out["peak_GBps"] = peak
    out["peak_kind"] = kind
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for name in (sys.argv[1:] or ["C2", "C3", "C4", "C5"]):
        run(name)
