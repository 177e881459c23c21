timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sort_fixup or degenerate" > gpurun_out/fix.log 2>&1; tail -15 gpurun_out/fix.log
