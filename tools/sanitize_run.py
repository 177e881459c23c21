"""Small evaluations covering every kernel, for compute-sanitizer memcheck/racecheck/synccheck:
all modes, p on the tcgen05 / CUDA-core / direct-pair M2L paths, both M2L summation modes, the
distinct target/source entry point and a 2-rank in-process distributed group."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from fmm_inputs import make_particles
from paper_1108_5815_b200 import FMM
from paper_1108_5815_b200.fmm import LocalGroup

COST = (2e-12, 6e-11, 2.5e-9)
cases = [("uniform", 3000, 10, 0.4, 64), ("mixed", 5000, 8, 0.45, 8), ("plummer", 4000, 13, 0.5, 32),
         ("uniform", 1000, 4, 0.5, 16), ("plummer", 3000, 12, 0.5, 24)]
for dist, n, p, th, nc in cases:
    xyz, q = make_particles(n, dist, 5)
    X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
    f = FMM(p=p, theta=th, ncrit=nc, tune=False)
    f.set_cost_model(*COST)
    for det in (True, False):
        f.set_deterministic(det)
        for mode in ("fmm", "treecode", "hybrid", "direct"):
            f.set_mode(mode)
            phi, grad = f.evaluate(X, Q)
            torch.cuda.synchronize()
            print(dist, n, p, mode, det, float(phi.abs().sum()), flush=True)
    f.set_mode("hybrid")
    phi, grad = f.evaluate_ts(X[: n // 3].contiguous(), X[n // 3:].contiguous(), Q[n // 3:].contiguous())
    torch.cuda.synchronize()
    f.close()

# rotation-based M2L (m2l_rot.cu), both summation modes
xyz, q = make_particles(4000, "plummer", 8)
X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
for pp in (6, 14):
    f = FMM(p=pp, theta=0.5, ncrit=24, tune=False)
    f.set_m2l_scheme("rotation")
    f.set_cost_model(*COST)
    for det in (True, False):
        f.set_deterministic(det)
        phi, grad = f.evaluate(X, Q)
        torch.cuda.synchronize()
        print("rotation", pp, det, float(phi.abs().sum()), flush=True)
    f.close()

# Cartesian expansions (cart.cu): every operator, all modes
xyz, q = make_particles(5000, "plummer", 7)
X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
f = FMM(p=4, theta=0.5, ncrit=16, tune=False)
f.set_basis("cartesian")
f.set_cost_model(*COST)
for mode in ("fmm", "treecode", "hybrid"):
    f.set_mode(mode)
    phi, grad = f.evaluate(X, Q)
    torch.cuda.synchronize()
    print("cartesian", mode, float(phi.abs().sum()), flush=True)
f.close()

# traversal overflow-and-retry paths (stack / list scratch and list buffers far too small, small
# theta = long lists): the retried traversal must not read past any buffer
os.environ["FMM_TRAV_CAP"] = "32"
os.environ["FMM_TRAV_LIST_EST"] = "2"
xyz, q = make_particles(40000, "plummer", 6)
f = FMM(p=4, theta=0.15, ncrit=16, tune=False)
f.set_cost_model(*COST)
f.set_mode("hybrid")
phi, grad = f.evaluate(torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda())
torch.cuda.synchronize()
print("overflow retry", float(phi.abs().sum()), flush=True)
f.close()
del os.environ["FMM_TRAV_CAP"], os.environ["FMM_TRAV_LIST_EST"]

# two in-process ranks (the distributed path: split-bound allreduce, particle and LET exchanges)
xyz, q = make_particles(6000, "plummer", 9)
grp = LocalGroup(2)
parts = np.array_split(np.random.default_rng(0).permutation(6000), 2)


def rank(r):
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        f = FMM(p=8, theta=0.45, ncrit=32, tune=False, group=(grp, r))
        f.set_cost_model(*COST)
        f.evaluate(torch.from_numpy(xyz[parts[r]]).cuda(), torch.from_numpy(q[parts[r]]).cuda())
        s.synchronize()
        f.close()


th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
[t.start() for t in th]
[t.join() for t in th]
grp.close()
print("SANITIZE_DONE")
