"""Spherical vs Cartesian expansions (NEXT-2) at low order on the B200: time-to-solution of the
C2 recipe (1M uniform, theta = 0.4, ncrit = 64, hybrid, cost model measured per basis) for
p = 1..4, error against the oracle's sampled direct sum, and the automatic switch's choice.
One JSON line per (p, basis). Usage: basis_sweep.py [n]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from fmm_inputs import make_particles
from oracle import oracle as O
from paper_1108_5815_b200 import FMM

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
xyz, q = make_particles(n, "uniform", 2)
X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
s = np.random.default_rng(0).choice(n, 1024, replace=False)
d = O.direct(xyz, q, s)
for p in (1, 2, 3, 4):
    f = FMM(p=p, theta=0.4, ncrit=64, mode="hybrid", tune=False)
    f.set_basis("auto")
    choice, auto_ms = f.basis()
    for basis in ("spherical", "cartesian"):
        f.set_basis(basis)  # (re-tunes its cost model)
        for _ in range(3):
            f.evaluate(X, Q)
        torch.cuda.synchronize()
        ms = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            phi, grad = f.evaluate(X, Q)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        f.set_timing(True)
        f.evaluate(X, Q)
        st = f.stats()
        f.set_timing(False)
        ph = phi.cpu().numpy()[s].astype(np.float64)
        gr = grad.cpu().numpy()[s].astype(np.float64)
        print(json.dumps({"p": p, "basis": basis, "n": n, "ms": float(np.median(ms)),
                          "err_phi": O.rel_l2(ph, d[0]), "err_grad": O.rel_l2(gr, d[1]),
                          "ms_m2l": st["ms_m2l"], "ms_upward": st["ms_upward"],
                          "ms_downward": st["ms_downward"], "n_m2l": st["n_m2l"],
                          "auto_choice": choice, "auto_ms": auto_ms}), flush=True)
    f.close()
