import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from fmm_inputs import make_particles
from oracle import oracle as O
from paper_1108_5815_b200 import FMM
mode_env = sys.argv[1]
for dist, n, p, th, nc in [("shell", 8000, 5, 0.5, 20), ("shell", 8000, 8, 0.5, 20), ("uniform", 8000, 5, 0.5, 20), ("plummer", 8000, 5, 0.5, 20)]:
    xyz, q = make_particles(n, dist, 4)
    f = FMM(p=p, theta=th, ncrit=nc, mode="fmm", tune=False)
    phi, grad = f.evaluate(torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda())
    torch.cuda.synchronize()
    ref = O.fmm(xyz, q, p, th, nc, O.FMM, want_structure=False)
    ph = phi.cpu().numpy()
    err = np.abs(ph - ref.phi) / np.abs(ref.phi)
    print(mode_env, dist, p, "rel phi %.2e grad %.2e  max pointwise %.2e" % (O.rel_l2(ph, ref.phi), O.rel_l2(grad.cpu().numpy(), ref.grad), err.max()), flush=True)
    f.close()
