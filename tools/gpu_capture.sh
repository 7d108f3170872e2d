#!/bin/bash
# Run on the GPU box (gpurun -- 'bash tools/gpu_capture.sh'): tests, smoke, bench
# (both arms), kernel table, ncu launch lists and full captures of the main
# kernels.  The .ncu-rep files exceed gpurun's output limit, so each capture is
# exported on the box (raw metrics CSV + details page) and the report deleted;
# tools/raw_summary.py / tools/ncu_summary.py turn the exports into profiles/.
O=gpurun_out/capture
mkdir -p $O
cap() { name=$1; shift
  ncu --set full --clock-control none --import-source on -o /tmp/$name -f "$@" > $O/ncu_$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details > $O/${name}_details.txt 2>/dev/null
  rm -f /tmp/$name.ncu-rep; }
python -m pytest tests -m gpu -q -rP 2>&1 | tail -45 > $O/pytest_gpu.log
python __graft_entry__.py smoke > $O/smoke.log 2>&1
python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python tools/kernel_bench.py > $O/kernel_bench.jsonl 2> $O/kernel_bench.err
python tools/transfer_bench.py C2 C3 C4 C5 > $O/transfer.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-scaling --no-cpu-baseline > $O/ncu_bench.log 2>&1
STMG_HOSTLOOP=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file $O/C2_launches.csv python tools/profile_solve.py C2 > $O/ncu_C2.log 2>&1
cap updown_C2 -k regex:k_updown -s 5 -c 1 python tools/profile_solve.py C2
for c in C2 C3 C4 C5; do cap residual_$c -k regex:k_apply -s 1 -c 1 python tools/profile_residual.py $c; done
for c in C3 C5; do cap dst_$c -k regex:k_dst -c 2 python tools/profile_dst.py $c 1; done
