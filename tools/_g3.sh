O=gpurun_out/r02c
mkdir -p $O
cap() { name=$1; shift
  ncu --set full --clock-control none --import-source on -o /tmp/$name -f "$@" > $O/ncu_$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details > $O/${name}_details.txt 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv 2>/dev/null | gzip > $O/${name}_source.csv.gz
  rm -f /tmp/$name.ncu-rep; }
for c in C2 C3 C4 C5; do
cap rows_$c -k regex:k_apply -s 1 -c 1 python tools/profile_residual.py $c
done
