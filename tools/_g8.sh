O=gpurun_out/r02h
mkdir -p $O
python tools/ab.py "STMG_L2_F=0" "STMG_L2_F=2" "STMG_L2_F=3" "STMG_L2_F=0" -- C2 > $O/l2f_ab2.txt 2>&1
