#!/usr/bin/env python3
"""Full-size golden fixtures for BASELINE configs C2..C5 (G = 1) from the CPU
oracle (TEST INFRASTRUCTURE: generates tests/golden/full_<cfg>.npz).

For each config this runs the reference solve loop (mg.cpp:134-166: r0 =
||f - A u0||, V(1,1) cycles with omega_t = 1/2 and exact DG block solves, stop
at ||r_k|| <= 1e-8 ||r_0||) on the oracle at the BASELINE size and records

  * the iteration count, the full residual history and the stop margin
    |r_k/r_0 - eps| / eps of the last cycle,
  * a seeded sample of 32768 entries of the iterate after cycle 1, after
    cycle 2 and at convergence (indices stored, plus the first and last 64
    entries of the vector).

The GPU tests (tests/test_gpu_full_parity.py) compare the B200 solve against
these fixtures, so the oracle never runs on the GPU box.  Inputs are the same
seeded generator bench.py uses (seed 42, f stream 0, u0 stream 1 folded into
f for C2).

Usage: OMP_NUM_THREADS=8 python tools/make_golden.py C2 [C4 C3 C5]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

CONFIGS = {  # (p_t, dim, space_level, time_level, T, random_u0) -- BASELINE configs
    "C2": (1, 2, 6, 8, 1.0, True),
    "C3": (2, 2, 7, 12, 1.0, False),
    "C4": (1, 3, 5, 10, 1.0, False),
    "C5": (1, 2, 8, 11, 1.0, False),
}
SEED = 42
EPS = 1e-8
NSAMPLE = 32768


def sample_indices(n: int, cfg: str) -> np.ndarray:
    rng = np.random.default_rng(1411_0519 + int(cfg[1:]))
    idx = rng.choice(n, size=min(n, NSAMPLE), replace=False)
    edge = np.concatenate([np.arange(min(64, n)), np.arange(max(n - 64, 0), n)])
    return np.unique(np.concatenate([idx, edge])).astype(np.int64)


def run(cfg: str) -> dict:
    p, dim, sl, tl, T, ru0 = CONFIGS[cfg]
    t0 = time.time()
    h = O.Hierarchy(p, dim, sl, tl, t_final=T)
    f = O.make_inputs(h, SEED, random_u0=ru0)
    u = np.zeros_like(f)
    idx = sample_indices(f.size, cfg)
    r0 = h.residual_norm(0, u, f)
    hist = [r0]
    samples = {}
    it = 0
    for k in range(1, 251):
        tc = time.time()
        h.mg_cycle_inplace(0, u, f, 1, 1, 1, 0.5)
        rk = h.residual_norm(0, u, f)
        hist.append(rk)
        it = k
        print(f"[{cfg}] cycle {k}: r/r0 = {rk / r0:.3e} ({time.time() - tc:.1f} s)", flush=True)
        if k in (1, 2):
            samples[f"u{k}"] = u[idx].copy()
        if rk <= EPS * r0:
            break
    samples["u_final"] = u[idx].copy()
    margin = abs(hist[-1] / hist[0] - EPS) / EPS
    meta = dict(config=cfg, p_t=p, dim=dim, space_level=sl, time_level=tl, t_final=T,
                random_u0=ru0, seed=SEED, eps=EPS, iterations=it, converged=hist[-1] <= EPS * r0,
                stop_margin=margin, dofs=int(f.size), levels=len(h.levels),
                oracle_wall_s=time.time() - t0, omp_threads=os.environ.get("OMP_NUM_THREADS"),
                cycle="V(1,1) omega_t=0.5 exact blocks, mu-driven coarsening",
                generator="tools/make_golden.py (oracle/stmg_oracle.cpp)")
    out = os.path.join(ROOT, "tests", "golden", f"full_{cfg}.npz")
    np.savez_compressed(out, idx=idx, history=np.array(hist), meta=json.dumps(meta), **samples)
    print(json.dumps(meta), flush=True)
    return meta


if __name__ == "__main__":
    for c in sys.argv[1:] or ["C2"]:
        run(c)
