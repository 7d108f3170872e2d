"""Per-launch sequence of an ncu --csv metrics log (launch order, grid, duration):
attributes the time of one V-cycle to its level kernels.  usage: launch_seq.py CSV [first] [count]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
gi = h.index("Grid Size") if "Grid Size" in h else None
seq = {}
for r in data:
    d = seq.setdefault(int(r[ii]), {"name": r[ki].split("(")[0].replace("void ", ""), "grid": r[gi] if gi else ""})
    try:
        d[r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:
        pass
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
count = int(sys.argv[3]) if len(sys.argv) > 3 else 60
for i in sorted(seq)[first:first + count]:
    d = seq[i]
    print(f"{i:5d} {d['name'][:44]:44s} {d['grid']:>16s} {d.get('gpu__time_duration.sum', 0) / 1e3:9.2f} us")
