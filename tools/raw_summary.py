"""Key metrics per kernel from an exported `ncu --page raw --csv` file
(the .ncu-rep stays on the GPU box: it exceeds the gpurun_out size limit):
python tools/raw_summary.py file_raw.csv [...]"""
import csv
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from ncu_summary import KEYS  # noqa: E402

EXTRA = ["smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
         "lts__throughput.avg.pct_of_peak_sustained_elapsed",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__occupancy_limit_registers",
         "launch__occupancy_limit_shared_mem", "launch__waves_per_multiprocessor",
         "launch__shared_mem_per_block_dynamic",
         "sm__warps_active.avg.pct_of_peak_sustained_active"]

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    h, units, data = rows[0], rows[1], rows[2:]
    print("#", path)
    for r in data:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        name = name.replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        print("==", name)
        seen = set()
        for k in KEYS + EXTRA:
            if k in h and k not in seen:
                seen.add(k)
                i = h.index(k)
                print(f"   {k:72s} {r[i]:>18s} {units[i]}")
