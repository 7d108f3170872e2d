"""Shared-memory wavefronts per SASS instruction (actual vs ideal) from an ncu
source page: python tools/smem_hot.py report.ncu-rep [kernel_index]."""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None and r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and r:
        cur["rows"].append(r)
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
b = blocks[k]
h = b["hdr"]
iw, ii, isrc, ismp = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal"), \
    h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iw] or 0) for r in b["rows"])
toti = sum(float(r[ii] or 0) for r in b["rows"])
print(b["name"][:80], f"shared wavefronts {tot:.3g} ideal {toti:.3g}")
top = sorted(b["rows"], key=lambda r: -float(r[iw] or 0))[:25]
for r in top:
    print(f"{float(r[iw]):12.3g} {float(r[ii]):12.3g} smp={r[ismp]:>6s}  {r[isrc].strip()[:70]}")
