timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
CFGS="C2 C3 C4" STEPS=10 bash tools/ab_bench.sh "new:"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.json')):
    d=json.loads([x for x in open(f) if x.startswith('{')][-1])
    ph=d['phases_ms']; print(f.split('/')[-1], round(d['ms_per_step'],3), {k[3:]:round(v,3) for k,v in ph.items()})
PY
