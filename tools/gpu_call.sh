timeout 900 python -m pytest tests/test_gpu_rotation.py -x -q > gpurun_out/tck.log 2>&1; tail -2 gpurun_out/tck.log
timeout 900 python tools/p_ladder.py 1000000 10 11 12 13 14 15 > gpurun_out/p_ladder2.jsonl 2> gpurun_out/p_ladder.err
python -c "
import json
for l in open('gpurun_out/p_ladder2.jsonl'):
    d=json.loads(l); print(d['p'], d['scheme'], round(d['ms'],3), round(d['ms_m2l'],3), '%.2e %.2e'%(d['err_phi'], d['err_grad']))
"
