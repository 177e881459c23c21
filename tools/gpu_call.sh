timeout 900 python -m pytest tests/test_gpu_check.py -x -q > gpurun_out/parity.log 2>&1; tail -2 gpurun_out/parity.log
