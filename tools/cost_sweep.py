"""Sensitivity of the step time to the hybrid cost model (PAPER.md:130 kernel pre-calculation):
the handle's tuned (t_pp, t_mp, t_ml) with t_pp scaled, C4 by default; median of 5 steps.
Usage: cost_sweep.py [config] [scale ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from fmm_inputs import CONFIGS, make_particles

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
scales = [float(x) for x in sys.argv[2:]] or [0.5, 0.7, 1.0, 1.4, 2.0]
cfg = CONFIGS[name]
xyz, q = make_particles(cfg["n"], cfg["dist"], cfg["seed"])
X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
f = bench.make_handle(cfg, "hybrid", False)
c0 = f.cost_model()
for s in scales:
    f.set_cost_model(c0[0] * s, c0[1], c0[2])
    for _ in range(2):
        f.evaluate(X, Q)
    torch.cuda.synchronize()
    ms = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f.evaluate(X, Q)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    st = f.stats()
    print(json.dumps({"config": name, "t_pp_scale": s, "cost": [c0[0] * s, c0[1], c0[2]], "ms": float(np.median(ms)),
                      "p2p_pairs": st["p2p_pairs"], "n_m2l": st["n_m2l"], "n_p2p": st["n_p2p"]}), flush=True)
f.close()
