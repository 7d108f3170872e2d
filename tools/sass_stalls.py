"""Aggregate ncu SASS-page stall reasons per kernel (run here on a .ncu-rep)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
        continue
    if cur is not None:
        cur["rows"].append(r)
seen = set()
for b in blocks:
    if b["name"] in seen:
        continue
    seen.add(b["name"])
    h, data = b["rows"][0], b["rows"][1:]
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = collections.Counter()
    src = h.index("Source")
    top = []
    for r in data:
        if len(r) < len(h):
            continue
        s = 0.0
        for c in cols:
            v = float(r[h.index(c)] or 0)
            tot[c] += v
            s += v
        top.append((s, r[0], r[src][:70]))
    allv = sum(tot.values()) or 1
    print(b["name"][:90])
    print("   reasons:", [(k[6:], round(100 * v / allv, 1)) for k, v in tot.most_common(8)])
    for s, a, t in sorted(top, reverse=True)[:6]:
        print(f"   {100 * s / allv:5.1f}%  {t}")
