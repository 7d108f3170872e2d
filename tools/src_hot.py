"""Warp-stall samples per CUDA source line from an ncu report (needs -lineinfo and
--import-source on): python tools/src_hot.py report.ncu-rep [kernel_index] [top]."""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": [], "hdr": None}
        blocks.append(cur)
    elif cur is not None and r and cur["hdr"] is None and ("Source" in r):
        cur["hdr"] = r
    elif cur is not None and r and cur["hdr"] is not None:
        cur["rows"].append(r)
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top_n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
b = blocks[k]
h = b["hdr"]
ismp = [i for i, c in enumerate(h) if c.startswith("Warp Stall Sampling (All")][0]
isrc = h.index("Source")
iline = h.index("Line") if "Line" in h else 0
tot = sum(float(r[ismp] or 0) for r in b["rows"] if len(r) > ismp)
print(b["name"][:90], "samples", tot)
for r in sorted((r for r in b["rows"] if len(r) > ismp), key=lambda r: -float(r[ismp] or 0))[:top_n]:
    print(f"{100 * float(r[ismp] or 0) / tot:5.1f}%  L{r[iline]:>5s}  {r[isrc].strip()[:90]}")
