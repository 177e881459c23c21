#!/bin/bash
# Scratch entry point for one gpurun call (edited per experiment; tools/profile_r2final.sh is the
# reproducible evidence run): full GPU suite, the default bench line, C4 launch lists.
out=gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > $out/gputest.log 2>&1; tail -2 $out/gputest.log
timeout 900 python bench.py > $out/r2f_bench.json 2> $out/r2f_bench.err; tail -c 400 $out/r2f_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file $out/r2f_launches_bench_C4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    --no-extras > $out/r2f_bench_under_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --nvtx --nvtx-include "profiled/" --csv --log-file $out/r2f_launch_C4.csv \
    python tools/profile_run.py C4 hybrid > $out/r2f_launch_C4.log 2>&1
ls -la $out/r2f_*csv
