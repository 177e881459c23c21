"""Quick GPU sanity/timing run used during development (not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from fmm_inputs import make_particles
from paper_1108_5815_b200 import FMM
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
dist = sys.argv[2] if len(sys.argv) > 2 else "uniform"
xyz, q = make_particles(n, dist, 2)
X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
t = time.time(); f = FMM(p=10, theta=0.4, ncrit=64, mode="hybrid"); print("create+tune s", time.time() - t, "cost", f.cost_model(), flush=True)
f.set_timing(True)
for mode in ["fmm", "hybrid", "treecode"]:
    f.set_mode(mode)
    for it in range(3):
        torch.cuda.synchronize(); t = time.time()
        phi, grad = f.evaluate(X, Q); torch.cuda.synchronize()
        wall = time.time() - t
    s = f.stats()
    print(mode, "wall ms %.2f" % (wall * 1e3), {k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()}, flush=True)
    pp = s["p2p_pairs"]; print("  P2P Gpair/s %.1f  GFLOP/s(19/pair) %.0f ; M2L /s %.3g  GFLOP/s(64k) %.0f" % (pp / s["ms_p2p"] / 1e6, 19 * pp / s["ms_p2p"] / 1e6, s["n_m2l"] / max(s["ms_m2l"], 1e-9) * 1e3, 63888 * s["n_m2l"] / max(s["ms_m2l"], 1e-9) / 1e6))
