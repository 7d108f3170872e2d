O=gpurun_out/r02m
mkdir -p $O
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -x -k "row_band and (case0 or case6 or case9)" > $O/memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -x -k "row_band and (case0 or case9)" > $O/racecheck.log 2>&1
tail -5 $O/memcheck.log; tail -8 $O/racecheck.log
