timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_check.py tests/test_gpu_dist.py -x -q > gpurun_out/parity.log 2>&1; tail -2 gpurun_out/parity.log
