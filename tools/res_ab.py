"""Physical residual GB/s per library variant: python tools/res_ab.py lib1.so lib2.so -- C2 C4"""
import json
import os
import subprocess
import sys

i = sys.argv.index("--")
libs, cfgs = sys.argv[1:i], sys.argv[i + 1:]
for lib in libs:
    env = dict(os.environ)
    if lib != "default":
        env["STMG_LIB"] = lib
    r = subprocess.run([sys.executable, "tools/kernel_bench.py"] + cfgs, env=env, capture_output=True,
                       text=True)
    out = []
    for line in r.stdout.splitlines():
        try:
            d = json.loads(line)
        except ValueError:
            continue
        out.append((d["config"], round(d["residual_phys"]["avg_ms"] * 1e3, 1),
                    round(d["residual_phys"]["alg_GBps"])))
    print(os.path.basename(lib), out, r.stderr[-300:] if not out else "", flush=True)
