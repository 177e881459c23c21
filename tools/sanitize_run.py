"""Small evaluations covering every kernel, for compute-sanitizer memcheck/racecheck/synccheck."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from fmm_inputs import make_particles
from paper_1108_5815_b200 import FMM
cases = [("uniform", 3000, 10, 0.4, 64), ("mixed", 5000, 8, 0.45, 8), ("plummer", 4000, 13, 0.5, 32),
         ("uniform", 1000, 4, 0.5, 16)]
for dist, n, p, th, nc in cases:
    xyz, q = make_particles(n, dist, 5)
    X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
    f = FMM(p=p, theta=th, ncrit=nc, tune=False)
    f.set_cost_model(2e-12, 6e-11, 2.5e-9)
    for mode in ("fmm", "treecode", "hybrid", "direct"):
        f.set_mode(mode)
        phi, grad = f.evaluate(X, Q)
        torch.cuda.synchronize()
        print(dist, n, p, mode, float(phi.abs().sum()), flush=True)
    f.close()
print("SANITIZE_DONE")
