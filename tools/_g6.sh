O=gpurun_out/r02f
mkdir -p $O
for d in 1 0; do
echo "STMG_DST_DENSE=$d" >> $O/dst_dense_ab.txt
STMG_DST_DENSE=$d python tools/profile_dst.py C4 3 2>&1 | tail -2 >> $O/dst_dense_ab.txt
done
echo "solve A/B (tools/ab.py)" >> $O/dst_dense_ab.txt
python tools/ab.py "STMG_DST_V1=1" "STMG_DST_V1=0" >> $O/dst_dense_ab.txt 2>&1
