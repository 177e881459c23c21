"""GPU parity of the Cartesian Taylor expansions (cart.cu) through the C ABI
(fmm_set_basis) against the FP64 oracle running the same basis (oracle/cartesian.c) with the same
tree, lists and cost model; and the automatic basis switch (FMM_BASIS_AUTO)."""
import numpy as np
import pytest

from fmm_inputs import make_particles

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1108_5815_b200 import FMM, FmmError  # noqa: E402

COST = (2e-12, 6e-11, 2.5e-9)


def run(f, xyz, q):
    phi, grad = f.evaluate(torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda())
    torch.cuda.synchronize()
    return phi.cpu().numpy().astype(np.float64), grad.cpu().numpy().astype(np.float64)


CASES = [("uniform", 1000, 4, 0.5, 16, 1), ("plummer", 20000, 3, 0.5, 32, 2),
         ("mixed", 8000, 2, 0.45, 24, 3), ("shell", 6000, 1, 0.5, 20, 4),
         ("uniform", 30000, 4, 0.4, 64, 5)]


@pytest.mark.parametrize("mode", ["fmm", "treecode", "hybrid"])
@pytest.mark.parametrize("dist,n,p,theta,ncrit,seed", CASES)
def test_cartesian_matches_oracle(O, mode, dist, n, p, theta, ncrit, seed):
    xyz, q = make_particles(n, dist, seed)
    f = FMM(p=p, theta=theta, ncrit=ncrit, mode=mode, tune=False)
    try:
        f.set_basis("cartesian")
        assert f.basis()[0] == "cartesian"
        f.set_cost_model(*COST)
        phi, grad = run(f, xyz, q)
        lists = O.canonical_tasks(f.export_lists())
    finally:
        f.close()
    omode = {"fmm": O.FMM, "treecode": O.TREECODE, "hybrid": O.HYBRID}[mode]
    ref = O.fmm(xyz, q, p, theta, ncrit, omode, cost=COST, basis="cartesian")
    assert np.array_equal(lists, O.canonical_tasks(ref.tasks))
    ep, eg = O.rel_l2(phi, ref.phi), O.rel_l2(grad, ref.grad)
    assert ep < 1e-5 and eg < 1e-5, (ep, eg)


def test_cartesian_c1_accuracy_vs_direct(O):
    # BASELINE configs[0] (C1: N=1000, p=4, theta=0.5, ncrit=16) in the low-accuracy basis
    xyz, q = make_particles(1000, "uniform", 1)
    f = FMM(p=4, theta=0.5, ncrit=16, mode="hybrid", tune=False)
    f.set_basis("cartesian")
    f.set_cost_model(*COST)
    phi, grad = run(f, xyz, q)
    f.close()
    d = O.direct(xyz, q)
    assert O.rel_l2(phi, d[0]) < 2e-3 and O.rel_l2(grad, d[1]) < 2e-2


def test_auto_basis_switch(O):
    # the automatic switch times both bases on the synthetic tuning set and keeps the faster one;
    # the evaluation then matches the oracle in the chosen basis
    xyz, q = make_particles(20000, "uniform", 9)
    f = FMM(p=3, theta=0.5, ncrit=32, mode="hybrid", tune=False)
    try:
        f.set_basis("auto")
        name, ms = f.basis()
        assert ms["spherical"] > 0 and ms["cartesian"] > 0
        assert name == ("cartesian" if ms["cartesian"] < ms["spherical"] else "spherical")
        cost = f.cost_model()
        phi, grad = run(f, xyz, q)
    finally:
        f.close()
    ref = O.fmm(xyz, q, 3, 0.5, 32, O.HYBRID, cost=cost, basis=name)
    assert O.rel_l2(phi, ref.phi) < 1e-5 and O.rel_l2(grad, ref.grad) < 1e-5


def test_cartesian_limits():
    f = FMM(p=6, theta=0.5, ncrit=32, tune=False)
    try:
        with pytest.raises(FmmError, match="Cartesian"):
            f.set_basis("cartesian")
        f.set_basis("auto")  # p > 4: stays spherical
        assert f.basis()[0] == "spherical"
    finally:
        f.close()
