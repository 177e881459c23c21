"""Diagnose per-particle errors at C2: the GPU path (FMM_LIB selects the library) against the FP64
oracle's full evaluation with the same tree, lists and a fixed cost model. Prints the worst
particles (|dgrad| / rms|grad|), their |grad| / rms and nearest-neighbour distance."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from scipy.spatial import cKDTree

from fmm_inputs import CONFIGS, make_particles
from oracle import oracle as O
from paper_1108_5815_b200 import FMM

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
xyz, q = make_particles(cfg["n"], cfg["dist"], cfg["seed"])
f = FMM(p=cfg["p"], theta=cfg["theta"], ncrit=cfg["ncrit"], mode="hybrid", tune=False)
cost = (5.6e-13, 1.19e-10, 2.2e-10)
f.set_cost_model(*cost)
f.set_deterministic(True)
phi, grad = f.evaluate(torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda())
torch.cuda.synchronize()
phi = phi.cpu().numpy().astype(np.float64)
grad = grad.cpu().numpy().astype(np.float64)
ref = O.fmm(xyz, q, cfg["p"], cfg["theta"], cfg["ncrit"], O.HYBRID, cost=f.cost_model(), want_structure=False)
rms = float(np.sqrt(np.mean(np.sum(ref.grad ** 2, axis=1))))
dg = np.linalg.norm(grad - ref.grad, axis=1) / rms
gm = np.linalg.norm(ref.grad, axis=1) / rms
dp = np.abs(phi - ref.phi) / np.abs(ref.phi)
d, _ = cKDTree(xyz.astype(np.float64)).query(xyz.astype(np.float64), k=2)
print("lib", os.environ.get("FMM_LIB", "default"), "relL2 phi", O.rel_l2(phi, ref.phi), "grad", O.rel_l2(grad, ref.grad))
print("max dphi", dp.max(), "max dgrad/rms", dg.max())
for i in np.argsort(-dg)[:8]:
    print(f"  i={i} dgrad/rms={dg[i]:.3e} |g|/rms={gm[i]:.3e} rel={dg[i] / gm[i]:.3e} nn={d[i, 1]:.3e} x={xyz[i]}")
