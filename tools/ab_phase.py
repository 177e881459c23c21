"""A/B timing of the phases of one config for the library named by FMM_LIB (development tool):
median per-phase CUDA-event times over several evaluations with a fixed cost model, plus the
result saved for a cross-variant comparison. Usage: FMM_LIB=... ab_phase.py C2 hybrid out.npy"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from fmm_inputs import CONFIGS, make_particles
from paper_1108_5815_b200 import FMM

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
mode = sys.argv[2] if len(sys.argv) > 2 else "hybrid"
out = sys.argv[3] if len(sys.argv) > 3 else None
xyz, q = make_particles(cfg["n"], cfg["dist"], cfg["seed"])
X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
f = FMM(p=cfg["p"], theta=cfg["theta"], ncrit=cfg["ncrit"], mode=mode, tune=False)
f.set_cost_model(5.76e-13, 1.18e-10, 2.17e-10)  # bench-measured C2 table (fixed for A/B)
f.set_deterministic(False)
f.set_timing(True)
ph = {}
for it in range(40):
    phi, grad = f.evaluate(X, Q)
    torch.cuda.synchronize()
    if it >= 5:
        for k, v in f.stats().items():
            if k.startswith("ms_"):
                ph.setdefault(k, []).append(v)
s = f.stats()
med = {k: round(float(np.median(v)), 4) for k, v in ph.items()}
pp = s["p2p_pairs"]
print(os.path.basename(os.environ.get("FMM_LIB", "libfmm.so")), med,
      "p2p TFLOP/s(18/pair) %.2f" % (18 * pp / med["ms_p2p"] / 1e9), flush=True)
if out:
    np.save(out, np.concatenate([phi.cpu().numpy()[:, None], grad.cpu().numpy()], 1))
