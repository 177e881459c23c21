"""One warm-up + one profiled fmm_evaluate (NVTX range "profiled") of a config for ncu captures,
in bench.py's launch configuration: cost model measured at create (FMM_COST=t_pp,t_mp,t_ml fixes
it instead) and the M2L summed by L2 vector reductions (FMM_DET=1: the deterministic order)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fmm_inputs import CONFIGS, make_particles
from paper_1108_5815_b200 import FMM
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
mode = sys.argv[2] if len(sys.argv) > 2 else "hybrid"
xyz, q = make_particles(cfg["n"], cfg["dist"], cfg["seed"])
X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
p = int(os.environ.get("FMM_P", cfg["p"]))  # (an order other than the config's, e.g. the p ladder)
f = FMM(p=p, theta=cfg["theta"], ncrit=cfg["ncrit"], mode=mode, tune="FMM_COST" not in os.environ)
if "FMM_COST" in os.environ:  # a fixed cost model (else the one measured at create, as bench.py)
    f.set_cost_model(*map(float, os.environ["FMM_COST"].split(",")))
f.set_deterministic(os.environ.get("FMM_DET", "0") == "1")
f.evaluate(X, Q); torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profiled")
f.evaluate(X, Q); torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print(f.stats())
