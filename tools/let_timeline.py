"""Per-rank event timeline of the local-essential-tree exchange (NEXT-3): R ranks
as an in-process group on one GPU, the C4 recipe at a reduced size split evenly over the ranks,
timing on. For the sender-side exchange (default) each rank reports the exchange's device time on
its own stream (ms_let) and how far it ran past the end of the traversal it overlaps
(ms_let_exposed; 0 = hidden); for the receiver-driven one (FMM_LET=recv) the exchange follows the
traversal, its host time is ms_comm. One JSON line per (mode, R, rank).
Usage: let_timeline.py [n] [R ...]"""
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from fmm_inputs import make_particles
from paper_1108_5815_b200 import FMM
from paper_1108_5815_b200.fmm import LocalGroup

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
Rs = [int(x) for x in sys.argv[2:]] or [2, 4]
xyz, q = make_particles(n, "uniform", 4)
for mode in ("send", "recv"):
    os.environ["FMM_LET"] = mode
    for R in Rs:
        grp = LocalGroup(R)
        out = [None] * R

        def worker(r):
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                f = FMM(p=10, theta=0.4, ncrit=64, tune=False, group=(grp, r))
                f.set_cost_model(5.6e-13, 1.2e-10, 2.2e-10)
                lo, hi = r * n // R, (r + 1) * n // R
                x = torch.from_numpy(np.ascontiguousarray(xyz[lo:hi])).cuda()
                c = torch.from_numpy(np.ascontiguousarray(q[lo:hi])).cuda()
                f.evaluate(x, c)
                f.set_timing(True)
                f.evaluate(x, c)
                s.synchronize()
                out[r] = f.stats()
                f.close()

        th = [threading.Thread(target=worker, args=(r,)) for r in range(R)]
        [t.start() for t in th]
        [t.join() for t in th]
        grp.close()
        for r, st in enumerate(out):
            print(json.dumps({"let": mode, "R": R, "rank": r, "n": n,
                              **{k: st[k] for k in ("ms_total", "ms_traverse", "ms_let", "ms_let_exposed",
                                                    "ms_comm", "let_cells", "let_particles", "bytes_sent")}}),
                  flush=True)
