"""Work balance of the distributed partition (SURVEY §8(f) NEXT-3 question): R in-process ranks on
one GPU, per-rank targets, P2P pairs, M2L pairs, the cost-model work estimate, its max/mean, and
the local-essential-tree volume each rank receives. Usage: python tools/dist_balance.py"""
import os, sys, threading
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from fmm_inputs import make_particles
from paper_1108_5815_b200 import FMM
from paper_1108_5815_b200.fmm import LocalGroup
for dist, n in (("plummer", 2_000_000), ("uniform", 2_000_000)):
    xyz, q = make_particles(n, dist, 3)
    R = 4
    parts = np.array_split(np.random.default_rng(0).permutation(n), R)
    grp = LocalGroup(R); st = [None] * R
    def w(r):
        torch.cuda.set_device(0); s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            f = FMM(p=10, theta=0.4, ncrit=64, tune=False, group=(grp, r))
            f.set_cost_model(5.76e-13, 1.18e-10, 2.17e-10); f.set_deterministic(False)
            f.evaluate(torch.from_numpy(xyz[parts[r]]).cuda(), torch.from_numpy(q[parts[r]]).cuda())
            s.synchronize(); st[r] = f.stats(); f.close()
    th = [threading.Thread(target=w, args=(r,)) for r in range(R)]
    [t.start() for t in th]; [t.join() for t in th]; grp.close()
    work = [5.76e-13 * s["p2p_pairs"] + 2.17e-10 * s["n_m2l"] + 1.18e-10 * s["m2p_evals"] for s in st]
    print(dist, "particles", [s["rank_hi"] - s["rank_lo"] for s in st], "p2p_pairs", [s["p2p_pairs"] for s in st],
          "m2l", [s["n_m2l"] for s in st], "work ms", [round(x * 1e3, 2) for x in work],
          "imbalance max/mean %.3f" % (max(work) / np.mean(work)), "let", [(s["let_cells"], s["let_particles"]) for s in st], flush=True)
