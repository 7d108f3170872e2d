O=gpurun_out/r02g
mkdir -p $O
for c in C3 C5 C4 C2; do
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${c}_launches.csv python tools/profile_solve.py $c > $O/ncu_$c.log 2>&1
done
