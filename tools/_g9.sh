O=gpurun_out/r02i
mkdir -p $O
for v in "" paper_1411_0519_b200/_variant_b256.so paper_1411_0519_b200/_variant_b256m3.so; do
echo "STMG_LIB=$v" >> $O/dst9_ab.txt
STMG_LIB=$v python tools/profile_dst.py C5 3 2>&1 | tail -2 >> $O/dst9_ab.txt
done
STMG_LIB=paper_1411_0519_b200/_variant_b256.so python -m pytest tests/test_gpu_parity.py -q -k "row_band or one_pass or operators" 2>&1 | tail -2 >> $O/dst9_ab.txt
