"""One warm-up + one profiled fmm_evaluate of the bench workload (C2) for ncu captures.
Uses a fixed B200 cost model (as measured by fmm_create) so no tuning kernels pollute the list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fmm_inputs import CONFIGS, make_particles
from paper_1108_5815_b200 import FMM
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
mode = sys.argv[2] if len(sys.argv) > 2 else "hybrid"
xyz, q = make_particles(cfg["n"], cfg["dist"], cfg["seed"])
X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
f = FMM(p=cfg["p"], theta=cfg["theta"], ncrit=cfg["ncrit"], mode=mode, tune=False)
cm = os.environ.get("FMM_COST", "1.29e-12,4.07e-10,7.67e-09").split(",")
f.set_cost_model(*map(float, cm))
f.evaluate(X, Q); torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profiled")
f.evaluate(X, Q); torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print(f.stats())
