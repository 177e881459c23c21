#!/bin/bash
# Scratch entry point for one gpurun call (edited per experiment; tools/profile_r2final.sh is the
# reproducible evidence run): M2L parity suites, then A/B of the fused key pass.
L=paper_1108_5815_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rotation.py tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
CFGS="C2 C4" tools/ab_bench.sh "new:" "old:FMM_LIB=$L/libfmm_old.so" "new2:" "old2:FMM_LIB=$L/libfmm_old.so"
python tools/ab_show.py 'gpurun_out/ab_*.json'
