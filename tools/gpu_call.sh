L=$PWD/paper_1108_5815_b200
FMM_LIB=$L/libfmm_lr2.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size or hybrid" > gpurun_out/parity.log 2>&1; tail -2 gpurun_out/parity.log
CFGS="C2 C3 C4" STEPS=10 bash tools/ab_bench.sh "base:" "lr2:FMM_LIB=$L/libfmm_lr2.so" "base2:" "lr2b:FMM_LIB=$L/libfmm_lr2.so"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.json')):
    try: d=json.loads([x for x in open(f) if x.startswith('{')][-1])
    except Exception: print(f,'FAIL'); continue
    ph=d['phases_ms']; print(f.split('/')[-1], round(d['ms_per_step'],3), 'p2p', round(ph['ms_p2p'],3), 'kernel', round(ph['ms_p2p_kernel'],3))
PY
