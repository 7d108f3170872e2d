O=gpurun_out/r02k
mkdir -p $O
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $O/pytest_gpu2.log
python tools/ab.py "STMG_X=0" -- C1 C2 C3 C4 C5 > $O/solve2.txt 2>&1
python bench.py --no-scaling --no-cpu-baseline > $O/bench_quick.json 2> $O/bench_quick.err
