L=$PWD/paper_1108_5815_b200
for v in base new pm4; do
  lib=$L/libfmm.so; [ $v != new ] && lib=$L/libfmm_$v.so
  for c in C2 C3 C4; do
    FMM_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "profiled/" -k regex:"k_l2p" --csv python tools/profile_run.py $c hybrid > gpurun_out/l2p_${v}_$c.csv 2>&1
    echo $v $c $(grep -h "k_l2p" gpurun_out/l2p_${v}_$c.csv | awk -F'","' '{print $NF}')
  done
done
FMM_LIB=$L/libfmm.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size or hybrid" > gpurun_out/parity.log 2>&1; tail -1 gpurun_out/parity.log
