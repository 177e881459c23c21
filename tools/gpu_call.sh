#!/bin/bash
# Scratch entry point for one gpurun call (edited per experiment; tools/profile_r2final.sh is the
# reproducible evidence run): the checked build three times, the full GPU suite, smoke(), bench.
out=gpurun_out
for k in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_check.py -m gpu -x -q > $out/chk_$k.log 2>&1; tail -n 1 $out/chk_$k.log; done
timeout 1800 python -m pytest tests -m gpu -x -q > $out/gputest.log 2>&1; tail -n 2 $out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1; tail -n 1 $out/smoke.log
timeout 900 python bench.py > $out/r2f_bench.json 2> $out/r2f_bench.err; tail -c 300 $out/r2f_bench.json
