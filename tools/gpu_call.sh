L=$PWD/paper_1108_5815_b200
FMM_LIB=$L/libfmm_rot.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size or hybrid" > gpurun_out/parity.log 2>&1; tail -2 gpurun_out/parity.log
CFGS="C2 C3 C4" STEPS=10 bash tools/ab_bench.sh "base:" "rot:FMM_LIB=$L/libfmm_rot.so" "base2:" "rot2:FMM_LIB=$L/libfmm_rot.so"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.json')):
    d=json.loads([x for x in open(f) if x.startswith('{')][-1])
    ph=d['phases_ms']; r=d['roofline']; fr = r['frac'] if r['kernel']=='k_p2p_tma' else r['secondary']['frac']
    print(f.split('/')[-1], round(d['ms_per_step'],3), 'kernel', round(ph['ms_p2p_kernel'],3), 'frac', round(fr,4))
PY
