#!/bin/bash
# Round-2 final evidence in one GPU call (writes gpurun_out/r2f_*):
#  * bench.py default run (C4 headline + C2/C3/deterministic extras) -- the JSON line
#  * ncu --set full of the P2P (k_p2p_tma) at C2 and C4 and of the M2L class GEMM (k_m2l_tc) at C2
#    and of the K-tiled tensor-core M2L (k_m2l_tck) at p = 12 on the C2 particles
#  * the launch list of bench.py's timed steps at C4 (NVTX "timed/"), kernel shares
#  * one C2 / C4 evaluation launch list with DRAM bytes (HBM GB/s per SURVEY §8(a) row)
out=gpurun_out
timeout 900 python bench.py > $out/r2f_bench.json 2> $out/r2f_bench.err
for cfg in C2 C4; do
  timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "profiled/" \
      -k regex:"k_p2p_tma" -c 1 -o $out/r2f_p2p_$cfg python tools/profile_run.py $cfg hybrid > $out/r2f_p2p_$cfg.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "profiled/" \
    -k regex:"k_m2l_tc<" --launch-skip 5 -c 1 -o $out/r2f_m2l_C2 python tools/profile_run.py C2 hybrid > $out/r2f_m2l_C2.log 2>&1
FMM_P=12 timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "profiled/" \
    -k regex:"k_m2l_tck" -c 1 -o $out/r2f_tck_p12 python tools/profile_run.py C2 hybrid > $out/r2f_tck_p12.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file $out/r2f_launches_bench_C4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    --no-extras > $out/r2f_bench_under_ncu.log 2>&1
for cfg in C2 C4; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --nvtx --nvtx-include "profiled/" --csv --log-file $out/r2f_launch_$cfg.csv \
      python tools/profile_run.py $cfg hybrid > $out/r2f_launch_$cfg.log 2>&1
done
ls -la $out/r2f_*
