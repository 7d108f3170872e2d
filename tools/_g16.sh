O=gpurun_out/r02p
mkdir -p $O
STMG_DST2D_PLANES=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_parity.py -q -x -k "n63 or operators or C4 or vcycle_iterates" 2>&1 | tail -3 > $O/pytest.log
for v in 0 1; do echo "STMG_DST2D_PLANES=$v" >> $O/planes_ab.txt; STMG_DST2D_PLANES=$v python tools/profile_dst.py C4 3 2>&1 | tail -2 >> $O/planes_ab.txt; done
python tools/ab.py "STMG_DST2D_PLANES=0" "STMG_DST2D_PLANES=1" -- C4 >> $O/planes_ab.txt 2>&1
