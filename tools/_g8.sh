O=gpurun_out/r02h
mkdir -p $O
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $O/pytest_gpu.log
python tools/ab.py "STMG_DST_V1=1" "STMG_DST_V1=0" -- C2 C3 C4 C5 > $O/solve_ab.txt 2>&1
