O=gpurun_out/r02e
mkdir -p $O
cap() { name=$1; shift
  ncu --set full --clock-control none --import-source on -o /tmp/$name -f "$@" > $O/ncu_$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details > $O/${name}_details.txt 2>/dev/null
  rm -f /tmp/$name.ncu-rep; }
python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
for c in C2 C3 C4 C5; do
cap residual_$c -k regex:k_apply -s 1 -c 1 python tools/profile_residual.py $c
done
cap smooth_C2 -s 12 -c 8 python tools/profile_smooth.py C2
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/smooth_C2_launches.csv python tools/profile_smooth.py C2 > $O/ncu_smooth_l.log 2>&1
python tools/kernel_bench.py > $O/kernel_bench.jsonl 2> $O/kernel_bench.err
