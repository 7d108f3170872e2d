"""A/B timing of full solves under different environments (one subprocess per
variant, so STMG_LIB / STMG_* switches apply from library load).

  python tools/ab.py "STMG_COARSE=0" "STMG_COARSE=1" -- C2 C5
Prints min / mean device ms per solve (device loop, no profiling) per variant.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys
sys.path.insert(0, %r)
from bench import CONFIGS, SEED
from paper_1411_0519_b200 import stmg
from paper_1411_0519_b200 import _capi as A
out = {}
for name in sys.argv[1:]:
    cfg = CONFIGS[name]
    h = stmg.Hierarchy(cfg["p_t"], cfg["dim"], cfg["space_level"], cfg["time_level"], cfg["t_final"])
    f, u = h.vector(0), h.vector(0)
    h.fill_uniform(f, SEED, 0)
    cc = stmg.CycleConfig(nu1=1, nu2=1)
    ts = []
    for k in range(8):
        A.check(A.lib().stmg_memset_zero(h._ctx, u.ptr, u.n * 8))
        rep = h.solve(f, u, cc, 1e-8)
        if k >= 3:
            ts.append(rep.device_time_seconds * 1e3)
    out[name] = [min(ts), sum(ts) / len(ts), rep.iterations]
    h.close()
print("RESULT " + json.dumps(out))
''' % ROOT


def main():
    i = sys.argv.index("--")
    variants, configs = sys.argv[1:i], sys.argv[i + 1:]
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            k, val = kv.split("=", 1)
            env[k] = val
        r = subprocess.run([sys.executable, "-c", CHILD] + configs, env=env, capture_output=True,
                           text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        print(v, json.loads(line[0][7:]) if line else ("FAILED", r.stderr[-500:]), flush=True)


if __name__ == "__main__":
    main()
