import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from fmm_inputs import make_particles
from paper_1108_5815_b200 import FMM
case = sys.argv[1]
f = FMM(p=4, theta=0.5, ncrit=8, tune=False, mode="fmm")
f.set_cost_model(2e-12, 6e-11, 2.5e-9)
if case == "zero":
    z = torch.zeros((0, 3), device="cuda"); print(f.evaluate(z, torch.zeros(0, device="cuda")))
elif case == "one":
    print(f.evaluate(torch.tensor([[0.1, 0.2, 0.3]], device="cuda"), torch.ones(1, device="cuda")))
elif case == "cluster":
    xyz = np.concatenate([np.full((37, 3), 0.25, np.float32), make_particles(29, "uniform", 3)[0]])
    X = torch.from_numpy(xyz).cuda(); Q = torch.ones(len(xyz), device="cuda")
    print(f.evaluate(X, Q)[0][:4]); print(f.stats())
elif case == "nonfinite":
    xyz = make_particles(100, "uniform", 1)[0]; xyz[5, 2] = np.inf
    try:
        f.evaluate(torch.from_numpy(xyz).cuda(), torch.ones(100, device="cuda"))
    except Exception as e:
        print("raised", e)
elif case == "host":
    x_h = torch.zeros((10, 3))
    print("rc", f.L.fmm_evaluate(f.h, x_h.data_ptr(), x_h.data_ptr(), 10, x_h.data_ptr(), x_h.data_ptr()))
torch.cuda.synchronize()
print("OK", case)
