O=gpurun_out/r02b
mkdir -p $O
python -m pytest tests/test_gpu_parity.py -x -q -k "row_band or operators_match" 2>&1 | tail -15 > $O/pytest_rows.log
for cfg in 1 2 3; do STMG_ROWS_CFG=$cfg python -m pytest tests/test_gpu_parity.py -x -q -k "row_band" 2>&1 | tail -1 >> $O/pytest_rows.log; done
echo default > $O/res_bench.txt
python tools/res_bench.py C2 C3 C4 C5 2>&1 | tail -1 >> $O/res_bench.txt 
python tools/res_bench.py C2 C3 C4 C5 2>&1 | tail -1 >> $O/res_bench.txt 
for cfg in 0 1 2 3; do 
echo "CFG=$cfg" >> $O/res_bench.txt
STMG_ROWS_CFG=$cfg python tools/res_bench.py C2 C3 C4 C5 2>&1 | tail -1 >> $O/res_bench.txt
done
