"""GPU parity of the rotation-based O(p^3) M2L (m2l_rot.cu) and of the
auto-tuning across translation schemes (fmm_set_m2l_scheme / fmm_tune), through the C ABI against
the FP64 oracle's direct double-loop M2L (the plain definition of the operator)."""
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


@pytest.mark.parametrize("deterministic", [True, False])
@pytest.mark.parametrize("dist,n,p,theta,ncrit,mode", [
    ("uniform", 8000, 4, 0.5, 16, "fmm"), ("plummer", 20000, 8, 0.45, 32, "hybrid"),
    ("uniform", 30000, 10, 0.4, 64, "fmm"), ("mixed", 6000, 12, 0.5, 24, "hybrid"),
    ("plummer", 5000, 13, 0.5, 32, "fmm"), ("uniform", 4000, 15, 0.5, 32, "fmm")])
def test_rotation_scheme_matches_oracle(O, dist, n, p, theta, ncrit, mode, deterministic):
    xyz, q = make_particles(n, dist, 100 + p)
    f = FMM(p=p, theta=theta, ncrit=ncrit, mode=mode, tune=False)
    try:
        f.set_m2l_scheme("rotation")
        f.set_deterministic(deterministic)
        f.set_cost_model(*COST)
        assert f.m2l_scheme()[0] == "rotation"
        phi, grad = run(f, xyz, q)
        if deterministic:  # bit-reproducible
            phi2, grad2 = run(f, xyz, q)
            assert np.array_equal(phi, phi2) and np.array_equal(grad, grad2)
    finally:
        f.close()
    omode = {"fmm": O.FMM, "hybrid": O.HYBRID}[mode]
    ref = O.fmm(xyz, q, p, theta, ncrit, omode, cost=COST, want_structure=False)
    ep, eg = O.rel_l2(phi, ref.phi), O.rel_l2(grad, ref.grad)
    assert ep < 1e-5 and eg < 1e-5, (ep, eg)


def test_rotation_equals_tensor_core_scheme():
    # the same operator evaluated two ways on identical lists: FP32 rounding apart
    xyz, q = make_particles(60000, "plummer", 7)
    out = {}
    for scheme in ("tc", "rotation", "gemm"):
        f = FMM(p=10, theta=0.4, ncrit=64, mode="fmm", tune=False)
        f.set_m2l_scheme(scheme)
        out[scheme] = run(f, xyz, q)
        f.close()
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    for s in ("rotation", "gemm"):
        assert rel(out[s][0], out["tc"][0]) < 2e-6 and rel(out[s][1], out["tc"][1]) < 2e-6, s


def test_scheme_autotuning():
    # fmm_tune times the M2L phase with every scheme available at this order and keeps the fastest
    for p, avail in ((8, {"tc", "gemm", "rotation", "pairs"}), (14, {"rotation", "pairs"})):
        f = FMM(p=p, theta=0.5, ncrit=32, mode="hybrid", tune=True)
        try:
            name, ms = f.m2l_scheme()
            measured = {k for k, v in ms.items() if v > 0}
            assert measured == avail, (p, ms)
            assert name == min(measured, key=lambda k: ms[k])
        finally:
            f.close()
    f = FMM(p=14, theta=0.5, ncrit=32, tune=False)
    with pytest.raises(FmmError, match="not available"):
        f.set_m2l_scheme("tc")
    f.close()


@pytest.mark.parametrize("p", [11, 12, 13, 14, 15])
def test_high_order_converges(O, p):
    # PAPER.md:205 runs p = 5..15: the default (tuned) scheme at p = 11..15 against the direct sum
    xyz, q = make_particles(6000, "uniform", 3)
    f = FMM(p=p, theta=0.5, ncrit=32, mode="fmm", tune=True)
    phi, grad = run(f, xyz, q)
    f.close()
    d = O.direct(xyz, q)
    assert O.rel_l2(phi, d[0]) < 3e-6 * 0.5 ** (p - 11) + 2e-7
