O=gpurun_out/r02l
mkdir -p $O
python tools/batch_trace.py 10 zero > $O/batch_trace_zero.txt 2>&1
