"""Pins of the oracle's Cartesian Taylor expansions (oracle/cartesian.c; SURVEY §8(f) NEXT-2,
PAPER.md:60 "capability to switch to Cartesian expansions", reading R17) against
things other than the oracle itself: closed-form derivatives of 1/r, finite differences, the
harmonicity of 1/r, exact polynomial shift identities, the point-charge closed form, brute-force
direct sums and convergence in the order p."""
import numpy as np
import pytest

from fmm_inputs import make_particles


def test_multi_index_enumeration(O):
    for p in range(0, 7):
        k3 = O.cart_multi(p)
        assert len(k3) == (p + 1) * (p + 2) * (p + 3) // 6 == O.cart_count(p)
        assert len({tuple(k) for k in k3.tolist()}) == len(k3)
        assert np.all(k3.sum(1) <= p) and np.all(np.diff(k3.sum(1)) >= 0)
        for i, (kx, ky, kz) in enumerate(k3.tolist()):
            assert O.cart_index(kx, ky, kz) == i


def test_derivative_tensor_closed_forms(O):
    d = np.array([0.31, -0.72, 1.13])
    x, y, z = d
    r = np.linalg.norm(d)
    a = O.cart_derivs(d, 4)
    ix = O.cart_index
    # a_k = (1/k!) d^k (1/r)
    assert np.isclose(a[ix(0, 0, 0)], 1 / r, rtol=1e-14)
    assert np.isclose(a[ix(1, 0, 0)], -x / r ** 3, rtol=1e-14)
    assert np.isclose(a[ix(0, 0, 1)], -z / r ** 3, rtol=1e-14)
    assert np.isclose(a[ix(2, 0, 0)], (3 * x * x - r * r) / r ** 5 / 2, rtol=1e-13)
    assert np.isclose(a[ix(1, 1, 0)], 3 * x * y / r ** 5, rtol=1e-13)
    assert np.isclose(a[ix(1, 1, 1)], -15 * x * y * z / r ** 7, rtol=1e-13)
    assert np.isclose(a[ix(3, 0, 0)], (-15 * x ** 3 / r ** 7 + 9 * x / r ** 5) / 6, rtol=1e-13)


def test_derivative_tensor_finite_differences_and_harmonicity(O):
    d = np.array([-0.45, 0.38, 0.91])
    P = 7
    a = O.cart_derivs(d, P)
    k3 = O.cart_multi(P)
    h = 1e-5
    for i, k in enumerate(k3.tolist()):
        s = sum(k)
        if 1 <= s:
            ax = int(np.argmax(k))  # an axis with k_ax >= 1
            m = list(k)
            m[ax] -= 1
            e = np.zeros(3)
            e[ax] = h
            fd = (O.cart_derivs(d + e, P)[O.cart_index(*m)] - O.cart_derivs(d - e, P)[O.cart_index(*m)]) / (2 * h)
            assert np.isclose(fd, k[ax] * a[i], rtol=1e-6, atol=1e-9 * abs(a).max()), k
        if s <= P - 2:  # 1/r is harmonic: sum_a (k_a + 1)(k_a + 2) a_{k + 2 e_a} = 0
            lap = 0.0
            for ax in range(3):
                m = list(k)
                m[ax] += 2
                lap += (k[ax] + 1) * (k[ax] + 2) * a[O.cart_index(*m)]
            assert abs(lap) < 1e-12 * abs(a).max(), k


def test_m2m_exact_shift(O):
    rng = np.random.default_rng(1)
    p = 5
    y = rng.random((40, 3)) * 0.5  # the child cell [0, .5)^3, centre .25
    q = rng.uniform(-1, 1, 40)
    cc = np.full(3, 0.25)
    cp = np.full(3, 0.5)
    Mc = O.cart_p2m(p, cc, y, q)
    direct = O.cart_p2m(p, cp, y, q)
    shifted = O.cart_m2m(p, Mc, cc - cp)
    assert np.allclose(shifted, direct, rtol=1e-13, atol=1e-15)


def test_l2l_exact_recentre(O):
    rng = np.random.default_rng(2)
    p = 5
    Lp = rng.standard_normal(O.cart_count(p))
    cp = np.array([0.5, 0.5, 0.5])
    cc = np.array([0.75, 0.25, 0.75])
    Lc = O.cart_l2l(p, Lp, cc - cp)
    x = cc + rng.uniform(-0.2, 0.2, (20, 3))
    a = O.cart_l2p(p, Lp, cp, x)
    b = O.cart_l2p(p, Lc, cc, x)
    assert np.allclose(a[0], b[0], rtol=1e-12) and np.allclose(a[1], b[1], rtol=1e-11)


def test_point_charge_at_centre(O):
    c = np.array([0.2, -0.1, 0.4])
    M = O.cart_p2m(4, c, c[None, :], np.array([2.5]))
    assert M[0] == 2.5 and np.all(M[1:] == 0)
    x = np.array([[1.3, 0.7, -0.9]])
    phi, grad = O.cart_m2p(4, M, c, x)
    d = x[0] - c
    r = np.linalg.norm(d)
    assert np.isclose(phi[0], 2.5 / r, rtol=1e-15)
    assert np.allclose(grad[0], -2.5 * d / r ** 3, rtol=1e-14)


def direct(xt, ys, qs):
    d = xt[:, None, :] - ys[None, :, :]
    r = np.linalg.norm(d, axis=2)
    return (qs / r).sum(1), -(qs[None, :, None] * d / r[:, :, None] ** 3).sum(1)


def test_m2p_converges_to_direct(O):
    rng = np.random.default_rng(3)
    c = np.zeros(3)
    y = rng.uniform(-0.5, 0.5, (50, 3))
    q = rng.uniform(-1, 1, 50)
    x = rng.uniform(-0.5, 0.5, (30, 3)) + np.array([2.5, 0.4, -0.3])
    ref = direct(x, y, q)
    errs = []
    for p in range(0, 9):
        phi, grad = O.cart_m2p(p, O.cart_p2m(p, c, y, q), c, x)
        errs.append(max(np.abs(phi - ref[0]).max() / np.abs(ref[0]).max(),
                        np.abs(grad - ref[1]).max() / np.abs(ref[1]).max()))
    assert all(b < a for a, b in zip(errs, errs[1:]))
    assert errs[-1] < 1e-5


def test_m2l_l2p_converges_to_direct(O):
    rng = np.random.default_rng(4)
    cs, ct = np.zeros(3), np.array([1.6, -1.2, 0.5])  # |d| = 2.06, cells of half-width 0.25
    y = rng.uniform(-0.25, 0.25, (60, 3))
    q = rng.uniform(-1, 1, 60)
    x = ct + rng.uniform(-0.25, 0.25, (40, 3))
    ref = direct(x, y, q)
    errs = []
    for p in range(1, 10):
        L = O.cart_m2l(p, O.cart_p2m(p, cs, y, q), ct - cs)
        phi, grad = O.cart_l2p(p, L, ct, x)
        errs.append(np.linalg.norm(phi - ref[0]) / np.linalg.norm(ref[0]))
    assert all(b < a for a, b in zip(errs, errs[1:]))
    assert errs[-1] < 1e-5


@pytest.mark.parametrize("mode", ["FMM", "HYBRID", "TREECODE"])
def test_whole_cartesian_fmm_converges(O, mode):
    # C1 (BASELINE configs[0]) with the Cartesian basis: relative L2 error against the direct
    # sum falls with p, and the spherical and Cartesian methods approach the same answer
    xyz, q = make_particles(1000, "uniform", 1)
    d = O.direct(xyz, q)
    m = getattr(O, mode)
    cost = (2e-12, 6e-11, 2.5e-9)
    errs = []
    for p in (1, 2, 4, 6):
        r = O.fmm(xyz, q, p, 0.5, 16, m, cost=cost, basis="cartesian")
        errs.append(O.rel_l2(r.phi, d[0]))
    assert all(b < a for a, b in zip(errs, errs[1:])), errs
    assert errs[2] < 2e-3  # p = 4, theta = 0.5: the low-accuracy regime Cartesian is for
    sph = O.fmm(xyz, q, 8, 0.5, 16, m, cost=cost)
    car = O.fmm(xyz, q, 8, 0.5, 16, m, cost=cost, basis="cartesian")
    assert O.rel_l2(car.phi, sph.phi) < 1e-5
    # same tree, same lists: only the expansions differ
    assert np.array_equal(O.canonical_tasks(car.tasks), O.canonical_tasks(sph.tasks))
