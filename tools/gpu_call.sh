#!/bin/bash
# Scratch entry point for one gpurun call (edited per experiment; tools/profile_r2final.sh is the
# reproducible evidence run): the GPU test suite and one bench line.
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.json
