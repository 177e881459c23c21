#!/bin/bash
# A/B of library variants on the GPU box: each env assignment list in "$@" runs bench.py once per
# config in $CFGS (default C2 C4); one JSON line per run in gpurun_out/ab_<tag>_<cfg>.json.
# usage: CFGS="C2 C4" tools/ab_bench.sh "new:" "old:FMM_P2P_LEGACY=1"
CFGS=${CFGS:-"C2 C4"}
STEPS=${STEPS:-10}
for spec in "$@"; do
  tag=${spec%%:*}; envs=${spec#*:}
  for cfg in $CFGS; do
    env $envs timeout 300 python bench.py --config $cfg --steps $STEPS --no-extras --no-cpu-baseline \
      > gpurun_out/ab_${tag}_${cfg}.json 2> gpurun_out/ab_${tag}_${cfg}.err
  done
done
