"""Summarise ncu output for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches <launches.csv>      # per-kernel shares
  python tools/ncu_summary.py full <report.ncu-rep>        # key raw metrics
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
    "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        try:
            v = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        name = name.replace("<unnamed>::", "")
        tot[name] += v
        cnt[name] += 1
    allt = sum(tot.values())
    out = [f"total kernel time {allt / 1e3:.1f} us over {sum(cnt.values())} launches "
           "(ncu: serialised, cold cache; compare shares)",
           f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k[:60]:60s} {cnt[k]:8d} {v / 1e3:10.1f} {v / 1e3 / cnt[k]:8.2f} {v / allt:6.3f}")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        name = name.replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        out.append(f"== {name}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"   {k:70s} {r[i]:>16s} {units[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else full(path))
