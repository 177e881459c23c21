timeout 1200 python -m pytest tests/test_gpu_check.py -x -q > gpurun_out/check.log 2>&1; tail -30 gpurun_out/check.log
