"""C2 p-ladder (PAPER.md:205 runs p = 5..15): for each order the handle is
created with the kernel pre-calculation, which also picks the M2L translation scheme (NEXT-1:
tensor-core class GEMM / CUDA-core class GEMM / rotation O(p^3) / per-pair); the line reports the
scheme, the M2L time each scheme measured during tuning, the time-to-solution (median of 10, CUDA
events, L2 warm) and the error against the oracle's direct sum on 1024 sampled targets.
Usage: p_ladder.py [n] [p ...]"""
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
ps = [int(x) for x in sys.argv[2:]] or list(range(4, 16))
xyz, q = make_particles(n, "uniform", 2)
X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
s = np.random.default_rng(0).choice(n, 1024, replace=False)
d = O.direct(xyz, q, s)
for p in ps:
    f = FMM(p=p, theta=0.4, ncrit=64, mode="hybrid", tune=False)
    f.set_deterministic(False)
    f.tune()
    scheme, sms = f.m2l_scheme()
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
    f.close()
    print(json.dumps({"p": p, "n": n, "scheme": scheme, "tuned_m2l_ms": sms, "ms": float(np.median(ms)),
                      "ms_m2l": st["ms_m2l"], "n_m2l": st["n_m2l"],
                      "phases_ms": {k: st[k] for k in ("ms_tree", "ms_upward", "ms_traverse", "ms_m2l",
                                                       "ms_p2p", "ms_m2p", "ms_downward")},
                      "err_phi": O.rel_l2(phi.cpu().numpy()[s].astype(np.float64), d[0]),
                      "err_grad": O.rel_l2(grad.cpu().numpy()[s].astype(np.float64), d[1])}), flush=True)
