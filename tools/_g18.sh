O=gpurun_out/r02r
mkdir -p $O
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $O/pytest_gpu.log
python tools/transfer_bench.py C2 C3 C4 C5 > $O/transfer2.jsonl 2>&1
