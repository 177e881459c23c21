L=$PWD/paper_1108_5815_b200
CFGS="C2 C3 C4" STEPS=10 bash tools/ab_bench.sh "new:" "old:FMM_LIB=$L/libfmm_old.so" "new2:" "old2:FMM_LIB=$L/libfmm_old.so"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.json')):
    d=json.loads([x for x in open(f) if x.startswith('{')][-1])
    ph=d['phases_ms']; print(f.split('/')[-1], round(d['ms_per_step'],3), 'up', round(ph['ms_upward'],3), 'down', round(ph['ms_downward'],3), 'trav', round(ph['ms_traverse'],3))
PY
