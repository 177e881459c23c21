CFGS="C2 C3 C4" STEPS=10 bash tools/ab_bench.sh "g8:" "g1:FMM_TREE_GRID=1" "g2:FMM_TREE_GRID=2" "g4:FMM_TREE_GRID=4"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.json')):
    try: d=json.loads([x for x in open(f) if x.startswith('{')][-1])
    except Exception: print(f,'FAIL'); continue
    ph=d['phases_ms']; print(f.split('/')[-1], round(d['ms_per_step'],3), 'tree', round(ph['ms_tree'],3))
PY
