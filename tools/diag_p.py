import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from fmm_inputs import make_particles
from oracle import oracle as O
from paper_1108_5815_b200 import FMM
xyz, q = make_particles(6000, "uniform", 3)
d = O.direct(xyz, q)
for p in (11, 12, 13, 14, 15):
    for sc in ("tc", "rotation", "pairs"):
        f = FMM(p=p, theta=0.5, ncrit=32, mode="fmm", tune=False)
        try:
            f.set_m2l_scheme(sc)
        except Exception as e:
            print(p, sc, 'n/a'); f.close(); continue
        phi, grad = f.evaluate(torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda())
        torch.cuda.synchronize()
        print(p, sc, O.rel_l2(phi.cpu().numpy().astype(np.float64), d[0]), O.rel_l2(grad.cpu().numpy().astype(np.float64), d[1]))
        f.close()
    f = FMM(p=p, theta=0.5, ncrit=32, mode="fmm", tune=True); print(p, 'tuned ->', f.m2l_scheme()); f.close()
