L=$PWD/paper_1108_5815_b200
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rotation.py tests/test_gpu_dist.py -x -q > gpurun_out/parity.log 2>&1; tail -2 gpurun_out/parity.log
CFGS="C2 C3 C4" STEPS=10 bash tools/ab_bench.sh "new:" "old:FMM_LIB=$L/libfmm_old.so" "new2:" "old2:FMM_LIB=$L/libfmm_old.so"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.json')):
    d=json.loads([x for x in open(f) if x.startswith('{')][-1])
    ph=d['phases_ms']; print(f.split('/')[-1], round(d['ms_per_step'],3), 'm2l', round(ph['ms_m2l'],3), 'trav', round(ph['ms_traverse'],3))
PY
