#!/bin/bash
# Round-2 profile evidence in one GPU call (writes gpurun_out/r2p_*):
#  * ncu --set full of the P2P and the M2L class GEMM at C2 and C4 (bench.py's launch configuration:
#    accumulate mode, cost model measured at create);
#  * the launch list of bench.py's timed steps at C4 (NVTX "timed/"), with DRAM bytes per launch;
#  * the launch list of one C2 and one C4 evaluation with DRAM bytes (HBM GB/s table per §8 row).
set -x
out=gpurun_out
for cfg in C2 C4; do
  ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "profiled/" \
      -k regex:"k_p2p_tma|k_m2l_tc" --launch-skip $([ $cfg = C2 ] && echo 5 || echo 7) -c 2 \
      -o $out/r2p_full_$cfg python tools/profile_run.py $cfg hybrid > $out/r2p_full_$cfg.log 2>&1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --nvtx --nvtx-include "profiled/" --csv --log-file $out/r2p_launch_$cfg.csv \
      python tools/profile_run.py $cfg hybrid > $out/r2p_launch_$cfg.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file $out/r2p_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    --no-extras > $out/r2p_bench_under_ncu.log 2>&1
