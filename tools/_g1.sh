set -x
O=gpurun_out/r02a
mkdir -p $O
cap() { # name, extra ncu args..., -- command
  name=$1; shift
  ncu --set full --clock-control none --import-source on -o /tmp/$name -f "$@" > $O/ncu_$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details > $O/${name}_details.txt 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv 2>/dev/null | gzip > $O/${name}_source.csv.gz
  rm -f /tmp/$name.ncu-rep
}
python -m pytest tests -m gpu -x -q -rP 2>&1 | tail -60 > $O/pytest_gpu.log
python __graft_entry__.py smoke > $O/smoke.log 2>&1
python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python tools/kernel_bench.py > $O/kernel_bench.jsonl 2> $O/kernel_bench.err
python tools/res_bench.py C2 C3 C4 C5 > $O/res_bench.txt 2>&1
for c in C2 C4; do
  cap residual_$c -k regex:k_apply -s 1 -c 1 python tools/profile_residual.py $c
done
for c in C2 C3 C4; do
  cap dst_$c -k regex:k_dst -c 3 python tools/profile_dst.py $c 1
done
cap smooth_C2 -s 12 -c 12 python tools/profile_smooth.py C2
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/smooth_C2_launches.csv python tools/profile_smooth.py C2 > $O/ncu_smooth_l.log 2>&1
du -sh $O; ls -la $O
