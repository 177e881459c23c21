import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from fmm_inputs import make_particles
from oracle import oracle as O
from paper_1108_5815_b200 import FMM
for n, p, dist in [(3000, 4, "uniform"), (20000, 10, "uniform"), (20000, 10, "plummer")]:
    xyz, q = make_particles(n, dist, 3)
    f = FMM(p=p, theta=0.5, ncrit=16, mode="fmm", tune=False)
    phi, grad = f.evaluate(torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda())
    torch.cuda.synchronize()
    ref = O.fmm(xyz, q, p, 0.5, 16, O.FMM, want_structure=False)
    print(n, p, dist, "rel phi", O.rel_l2(phi.cpu().numpy(), ref.phi), "grad", O.rel_l2(grad.cpu().numpy(), ref.grad), flush=True)
    f.close()
