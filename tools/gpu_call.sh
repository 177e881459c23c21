#!/bin/bash
# Scratch entry point for one gpurun call (edited per experiment; tools/profile_r2final.sh is the
# reproducible evidence run): M2L parity tests, then an A/B of the class sort's payload.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rotation.py tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
CFGS="C2 C3 C4" tools/ab_bench.sh "rec:" "idx:FMM_M2L_IDXSORT=1" "rec2:" "idx2:FMM_M2L_IDXSORT=1"
python tools/ab_show.py 'gpurun_out/ab_*.json' | tail -20
