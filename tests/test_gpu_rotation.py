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


@pytest.mark.parametrize("deterministic", [True, False])
@pytest.mark.parametrize("dist,n,p,theta,ncrit,mode", [
    ("uniform", 6000, 11, 0.5, 32, "fmm"), ("mixed", 6000, 12, 0.5, 24, "hybrid"),
    ("plummer", 5000, 13, 0.5, 32, "fmm"), ("uniform", 4000, 14, 0.5, 32, "fmm"),
    ("uniform", 4000, 15, 0.5, 32, "fmm"), ("plummer", 8000, 15, 0.45, 48, "hybrid")])
def test_ktiled_tensor_core_scheme_matches_oracle(O, dist, n, p, theta, ncrit, mode, deterministic):
    """10 < p <= 15: the K-tiled tcgen05 class GEMM (m2l_tc.cu k_m2l_tck: float-order operators
    streamed through shared memory in 32-column chunks, D in TMEM) against the oracle's direct
    double-loop M2L."""
    xyz, q = make_particles(n, dist, 200 + p)
    f = FMM(p=p, theta=theta, ncrit=ncrit, mode=mode, tune=False)
    try:
        f.set_m2l_scheme("tc")
        f.set_deterministic(deterministic)
        f.set_cost_model(*COST)
        assert f.m2l_scheme()[0] == "tc"
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


def test_ktiled_equals_rotation_scheme():
    # p = 13 on identical lists: the K-tiled tensor-core GEMM and the rotation scheme agree to
    # FP32 rounding
    xyz, q = make_particles(40000, "uniform", 9)
    out = {}
    for scheme in ("tc", "rotation"):
        f = FMM(p=13, theta=0.45, ncrit=48, mode="fmm", tune=False)
        f.set_m2l_scheme(scheme)
        out[scheme] = run(f, xyz, q)
        f.close()
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    assert rel(out["rotation"][0], out["tc"][0]) < 2e-6 and rel(out["rotation"][1], out["tc"][1]) < 2e-6


def test_scheme_autotuning():
    # fmm_tune times the M2L phase with every scheme available at this order and keeps the fastest
    for p, avail in ((8, {"tc", "gemm", "rotation", "pairs"}), (14, {"tc", "rotation", "pairs"})):
        f = FMM(p=p, theta=0.5, ncrit=32, mode="hybrid", tune=True)
        try:
            name, ms = f.m2l_scheme()
            measured = {k for k, v in ms.items() if v > 0}
            assert measured == avail, (p, ms)
            assert name == min(measured, key=lambda k: ms[k])
        finally:
            f.close()
    f = FMM(p=16, theta=0.5, ncrit=32, tune=False)
    with pytest.raises(FmmError, match="not available"):
        f.set_m2l_scheme("tc")
    f.close()


@pytest.mark.parametrize("p", [11, 12, 13, 14, 15])
def test_high_order_converges(O, p):
    # PAPER.md:205 runs p = 5..15: the default (tuned) scheme at p = 11..15 against the direct sum
    # The floor is the scheme's FP32 rounding: 2e-7 for the rotation and per-pair schemes (FP32
    # FMA chains), 6e-7 for the 3xTF32 tensor-core GEMM, whose FP32 accumulation runs inside the
    # tensor core over K = 2 nc products (measured 5.2e-7 at p = 11..15 with the rounded split and
    # FP64-built operators; truncation error 3e-6 * 2^-(p-11) on top).
    xyz, q = make_particles(6000, "uniform", 3)
    f = FMM(p=p, theta=0.5, ncrit=32, mode="fmm", tune=True)
    scheme = f.m2l_scheme()[0]
    phi, grad = run(f, xyz, q)
    f.close()
    d = O.direct(xyz, q)
    floor = 6e-7 if scheme == "tc" else 2e-7
    assert O.rel_l2(phi, d[0]) < 3e-6 * 0.5 ** (p - 11) + floor, scheme
