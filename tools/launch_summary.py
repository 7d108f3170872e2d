"""Per-kernel summary of an ncu --metrics CSV (duration and DRAM bytes)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ii, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "usecond": 1e3,
        "msecond": 1e6, "nsecond": 1}
per, names = collections.defaultdict(dict), {}
for r in data:
    try:
        v = float(r[vi].replace(",", ""))
    except (ValueError, IndexError):
        continue
    per[r[ii]][r[mi]] = v * mult.get(r[ui], 1)
    names[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "").replace("unnamed>::", "")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, d in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += d.get("dram__bytes_read.sum", 0)
    a[2] += d.get("dram__bytes_write.sum", 0)
    a[3] += d.get("gpu__time_duration.sum", 0)
tot = sum(a[3] for a in agg.values())
print(f"{sys.argv[1]}: ncu serialised launches (cold L2 per launch): compare shares, not absolutes")
print(f"{'kernel':38s} {'n':>5s} {'avg_us':>9s} {'share':>6s} {'rd_MB/l':>9s} {'wr_MB/l':>9s} {'dram_GB/s':>9s}")
for k, (n, rd, wr, t) in sorted(agg.items(), key=lambda x: -x[1][3]):
    print(f"{k[:38]:38s} {n:5d} {t / n / 1e3:9.2f} {t / tot:6.3f} {rd / n / 1e6:9.2f} {wr / n / 1e6:9.2f} "
          f"{(rd + wr) / t:9.1f}")
