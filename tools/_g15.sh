O=gpurun_out/r02o
mkdir -p $O
python -m pytest tests -m gpu -q -rP 2>&1 | tail -45 > $O/pytest_gpu.log
python __graft_entry__.py smoke > $O/smoke.log 2>&1
python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python tools/kernel_bench.py > $O/kernel_bench.jsonl 2> $O/kernel_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-scaling --no-cpu-baseline > $O/ncu_bench.log 2>&1
