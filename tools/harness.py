"""The reference's validation / scaling workflows on the GPU path
(bench.cpp:31-197):

  rho      two-grid factor measured on the GPU vs the LFA prediction over
           (p_t, mu, semi/full) -> profiles/r01_harness_rho.json
  weak     weak scaling in time (2 steps per "thread", tau fixed): MG solve
           time vs the sequential forward substitution, both on one GPU
           -> scaling CSV with the fwd_sub column (config.scaling_csv)
  strong   strong scaling over time-slab shards S = 1, 2, 4, 8 emulated on ONE
           GPU (virtual shards: same halo / gather / scatter driver as the
           multi-GPU path, not a multi-GPU measurement)

  python tools/harness.py rho|weak|strong|all [--out DIR]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0519_b200 import _capi as A  # noqa: E402
from paper_1411_0519_b200 import config, lfa, stmg  # noqa: E402


def rho_table():
    cfg = stmg.CycleConfig(nu1=1, nu2=1)
    rows = []
    for p in (0, 1, 2):
        for mu in (0.1, 0.3, 1.0, 3.0, 10.0, 100.0):
            for mode, name in ((lfa.SEMI, "semi"), (lfa.FULL, "full")):
                m = lfa.measure_convergence_factor(p, 1, 7, 6, mu, mode, cfg, seed=42,
                                                   n_theta_x=256, n_theta_t=256)
                rows.append({"p_t": p, "mu": mu, "mode": name, "measured": m.measured_rho,
                             "predicted": m.predicted_rho, "iterations": m.n_iterations_used,
                             "abs_diff": abs(m.measured_rho - m.predicted_rho)})
                print(json.dumps(rows[-1]), flush=True)
    return {"problem": "1D, space level 7 (255 nodes), 64 time steps, f = 0, random guess, "
                       "two-grid V(1,1), omega_t = 1/2, exact block solves",
            "acceptance": "|measured - predicted| <= 0.05 (SPEC.md:655)",
            "max_abs_diff": max(r["abs_diff"] for r in rows), "rows": rows}


def _solve_time(h, f, cc, eps=1e-8, reps=3):
    best, it = float("inf"), 0
    for _ in range(reps):
        u = h.vector(0)
        r = h.solve(f, u, cc, eps)
        best, it = min(best, r.device_time_seconds), r.iterations
    return best, it


def weak(p_t=1, dim=2, space_level=6, max_level=11):
    cc = stmg.CycleConfig(nu1=1, nu2=1)
    recs = []
    tau = 1.0 / 256
    for tl in range(1, max_level + 1):
        nt = 2 ** tl
        h = stmg.Hierarchy(p_t, dim, space_level, tl, t_final=tau * nt)
        f = h.vector(0)
        h.fill_uniform(f, 42, 0)
        t_mg, it = _solve_time(h, f, cc)
        u = h.vector(0)
        best = float("inf")
        for _ in range(4):  # the first call is warm-up
            h.synchronize()
            t0 = time.perf_counter()
            stmg.check(A.lib().stmg_forward_substitution(h._ctx, 0, f.ptr, u.ptr))
            h.synchronize()
            best = min(best, time.perf_counter() - t0) if _ else best
        recs.append(config.ScalingRecord(nt // 2, nt, h.levels[0]["n_x"], p_t, it, t_mg, best))
        h.close()
    return config.scaling_csv(recs, True)


def strong(p_t=1, dim=2, space_level=7, time_level=10):
    cc = stmg.CycleConfig(nu1=1, nu2=1)
    recs = []
    for S in (1, 2, 4, 8):
        h = stmg.Hierarchy(p_t, dim, space_level, time_level, shards=(S if S > 1 else 0))
        f = h.vector(0)
        h.fill_uniform(f, 42, 0)
        t_mg, it = _solve_time(h, f, cc)
        recs.append(config.ScalingRecord(S, 2 ** time_level, h.levels[0]["n_x"], p_t, it, t_mg))
        h.close()
    return config.scaling_csv(recs, False)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["rho", "weak", "strong", "all"])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = {}
    if a.what in ("rho", "all"):
        out["rho"] = rho_table()
    if a.what in ("weak", "all"):
        out["weak_csv"] = weak()
        print(out["weak_csv"], flush=True)
    if a.what in ("strong", "all"):
        out["strong_virtual_shards_csv"] = strong()
        print(out["strong_virtual_shards_csv"], flush=True)
    if a.out:
        os.makedirs(a.out, exist_ok=True)
        with open(os.path.join(a.out, f"harness_{a.what}.json"), "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
