#!/bin/bash
# Scratch entry point for one gpurun call (edited per experiment; tools/profile_r2final.sh is the
# reproducible evidence run): the GPU test suite, then the evidence run.
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
bash tools/profile_r2final.sh > /dev/null 2>&1
timeout 1500 python tools/config_sweep.py configs --steps 10 > gpurun_out/r2f_configs.jsonl 2> gpurun_out/r2f_configs.err
tail -c 300 gpurun_out/r2f_bench.json
