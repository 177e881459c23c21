L=$PWD/paper_1108_5815_b200
CFGS="C2 C3 C4" STEPS=10 bash tools/ab_bench.sh "base:" "ob976:FMM_LIB=$L/libfmm_ob976.so" "ob2s:FMM_LIB=$L/libfmm_ob2s1440.so"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.json')):
    d=json.loads([x for x in open(f) if x.startswith('{')][-1])
    ph=d['phases_ms']; print(f.split('/')[-1], round(d['ms_per_step'],3), 'kernel', round(ph['ms_p2p_kernel'],3))
PY
