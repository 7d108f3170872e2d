O=gpurun_out/r02n
mkdir -p $O
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $O/pytest_gpu.log
python tools/ab.py "STMG_UPDOWN_BLOCK=128" "STMG_UPDOWN_BLOCK=64" "STMG_UPDOWN_BLOCK=0" "STMG_UPDOWN_BLOCK=128" "STMG_UPDOWN_BLOCK=64" -- C2 > $O/block_ab.txt 2>&1
python tools/ab.py "STMG_UPDOWN_BLOCK=128" "STMG_UPDOWN_BLOCK=64" -- C4 C5 >> $O/block_ab.txt 2>&1
