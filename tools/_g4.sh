O=gpurun_out/r02d
mkdir -p $O
python -m pytest tests -m gpu -q -rP 2>&1 | tail -40 > $O/pytest_gpu.log
python tools/kernel_bench.py > $O/kernel_bench.jsonl 2> $O/kernel_bench.err
