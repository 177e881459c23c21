"""Live per-kernel GPU times (CUPTI via torch.profiler) of one fmm_evaluate of a config, with the
GPU idle time between kernels. Usage: kernel_times.py [C2] [hybrid] [top]"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from fmm_inputs import CONFIGS, make_particles
from paper_1108_5815_b200 import FMM

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
mode = sys.argv[2] if len(sys.argv) > 2 else "hybrid"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
xyz, q = make_particles(cfg["n"], cfg["dist"], cfg["seed"])
X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
f = FMM(p=cfg["p"], theta=cfg["theta"], ncrit=cfg["ncrit"], mode=mode)
f.set_deterministic(os.environ.get("FMM_DET", "0") == "1")
for _ in range(3):
    f.evaluate(X, Q)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    f.evaluate(X, Q)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
agg = defaultdict(lambda: [0.0, 0])
for e in evs:
    name = e.name.split("(")[0].replace("void ", "")
    if "cub::" in name:
        name = name.split("<")[0]
    agg[name][0] += e.time_range.elapsed_us()
    agg[name][1] += 1
busy = sum(v[0] for v in agg.values())
span = evs[-1].time_range.end - evs[0].time_range.start
print(f"{len(evs)} GPU activities, busy {busy:.0f} us, span {span:.0f} us, idle {span - busy:.0f} us")
for k, (us, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[:60]:60s} {us:8.1f} {n:4d}")
# largest gaps
gaps = []
for a, b in zip(evs, evs[1:]):
    gaps.append((b.time_range.start - a.time_range.end, a.name.split("(")[0][:40], b.name.split("(")[0][:40]))
gaps.sort(reverse=True)
print("largest idle gaps (us):")
for g in gaps[:12]:
    print(f"  {g[0]:7.1f}  after {g[1]}  before {g[2]}")
if os.environ.get("TIMELINE"):
    t0 = evs[0].time_range.start
    acc_idle = 0.0
    for a, b in zip(evs, evs[1:]):
        g = b.time_range.start - a.time_range.end
        acc_idle += max(g, 0)
        print(f"{a.time_range.start - t0:9.1f} {a.time_range.elapsed_us():8.1f}  gap {g:6.1f}  cum_idle {acc_idle:7.1f}  {a.name.split('(')[0][:50]}")
