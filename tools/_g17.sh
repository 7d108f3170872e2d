O=gpurun_out/r02q
mkdir -p $O
python tools/inexact_bench.py C2 C3 C4 > $O/inexact.jsonl 2>&1
STMG_BLOCK=vcycle STMG_HOSTLOOP=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/C2_inexact_launches.csv python tools/profile_solve.py C2 > $O/ncu.log 2>&1
