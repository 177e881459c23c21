"""Oracle pins: solid harmonics and the seven operators.

Every check is against something other than the oracle itself: scipy's associated Legendre
functions (closed form of R and I), 1/|x-y| (the Laplace expansion), point-charge closed forms,
brute-force direct sums, finite differences and exact translation identities.
"""
import math

import numpy as np
import pytest
from scipy.special import lpmv

rng = np.random.default_rng(1234)


def closed_R(x, n, m):
    r = np.linalg.norm(x)
    ct = x[2] / r if r > 0 else 1.0
    ph = math.atan2(x[1], x[0])
    am = abs(m)
    val = r ** n * lpmv(am, n, ct) * np.exp(1j * am * ph) / math.factorial(n + am)
    return val if m >= 0 else (-1) ** am * np.conj(val)


def closed_I(x, n, m):
    r = np.linalg.norm(x)
    ct = x[2] / r
    ph = math.atan2(x[1], x[0])
    am = abs(m)
    val = math.factorial(n - am) * lpmv(am, n, ct) * np.exp(1j * am * ph) / r ** (n + 1)
    return val if m >= 0 else (-1) ** am * np.conj(val)


@pytest.mark.parametrize("x", [[0.3, -0.2, 0.5], [-1.1, 0.7, -0.4], [0.0, 0.0, 0.8], [0.2, 0.1, 0.0]])
def test_harmonics_match_legendre_closed_form(O, x):
    P = 12
    x = np.array(x)
    R = O.harm_R(x, P)
    Iv = O.harm_I(x, P)
    for n in range(P + 1):
        for m in range(-n, n + 1):
            cr = closed_R(x, n, m)
            ci = closed_I(x, n, m)
            assert abs(R[O.idx(n, m)] - cr) <= 1e-12 * max(1.0, abs(cr)), (n, m)
            assert abs(Iv[O.idx(n, m)] - ci) <= 1e-12 * max(1.0, abs(ci)), (n, m)


def test_harmonics_axis_special_case(O):
    # On the z axis only m = 0 survives: R_n^0 = z^n / n!, I_n^0 = n! / z^(n+1).
    z = 0.7
    R = O.harm_R([0, 0, z], 8)
    Iv = O.harm_I([0, 0, z], 8)
    for n in range(9):
        assert R[O.idx(n, 0)] == pytest.approx(z ** n / math.factorial(n), rel=1e-14)
        assert Iv[O.idx(n, 0)] == pytest.approx(math.factorial(n) / z ** (n + 1), rel=1e-13)
        for m in range(1, n + 1):
            assert abs(R[O.idx(n, m)]) < 1e-15 and abs(Iv[O.idx(n, m)]) < 1e-15


def test_laplace_expansion_identity(O):
    # 1/|x-y| = sum conj(R_n^m(y)) I_n^m(x) for |y| < |x|; geometric convergence in P.
    x = np.array([1.3, -0.9, 0.6])
    y = np.array([0.2, 0.15, -0.1])
    P = 30
    s = np.sum(np.conj(O.harm_R(y, P)) * O.harm_I(x, P))
    assert abs(s.imag) < 1e-14
    assert s.real == pytest.approx(1.0 / np.linalg.norm(x - y), rel=1e-14)


# ---------------- P2M / M2P ----------------
def test_p2m_charge_at_centre(O):
    c = np.array([0.1, 0.2, 0.3])
    M = O.p2m(6, c, [c], [2.5])
    assert M[0] == pytest.approx(2.5)
    assert np.all(np.abs(M[1:]) == 0)


def test_p2m_neutral_symmetric_pair(O):
    c = np.zeros(3)
    M = O.p2m(6, c, [[0.1, 0.2, 0.3], [-0.1, -0.2, -0.3]], [1.0, -1.0])
    assert abs(M[0]) == 0.0


def test_m2p_monopole_is_point_charge(O):
    # a monopole source gives the exact point-charge potential and force.
    c = np.array([0.2, -0.1, 0.4])
    M = np.zeros(O.nterms(8), complex)
    M[0] = 3.0
    x = rng.normal(size=(5, 3)) + 3.0
    phi, grad = O.m2p(8, M, c, x)
    d = x - c
    r = np.linalg.norm(d, axis=1)
    np.testing.assert_allclose(phi, 3.0 / r, rtol=1e-14)
    np.testing.assert_allclose(grad, -3.0 * d / r[:, None] ** 3, rtol=1e-13)


def test_p2m_m2p_far_field_matches_direct(O):
    # random 10-particle cell evaluated at 5x radius, p=10 -> <= 1e-6 relative.
    c = np.zeros(3)
    y = rng.uniform(-0.5, 0.5, size=(10, 3))
    q = rng.uniform(0.1, 1.0, 10)
    M = O.p2m(10, c, y, q)
    x = rng.normal(size=(20, 3))
    x = 5.0 * np.sqrt(3) * 0.5 * x / np.linalg.norm(x, axis=1)[:, None]
    phi, grad = O.m2p(10, M, c, x)
    pd, gd = O.p2p(x, y, q)
    assert np.max(np.abs(phi - pd) / np.abs(pd)) < 1e-6
    assert np.linalg.norm(grad - gd) / np.linalg.norm(gd) < 1e-5


# ---------------- M2M / L2L (exact identities) ----------------
def test_m2m_zero_shift_identity(O):
    M = rng.normal(size=O.nterms(7)) + 1j * rng.normal(size=O.nterms(7))
    np.testing.assert_allclose(O.m2m(7, M, [0, 0, 0]), M, rtol=0, atol=1e-15)


def test_m2m_exact_chain_vs_direct_p2m(O):
    # R addition theorem: P2M(parent) == sum_children M2M(P2M(child)) to round-off.
    p = 10
    cp = np.array([0.5, 0.5, 0.5])
    Mp_direct = np.zeros(O.nterms(p), complex)
    Mp_chain = np.zeros(O.nterms(p), complex)
    for o in range(8):
        off = np.array([(o >> 2) & 1, (o >> 1) & 1, o & 1]) - 0.5
        cc = cp + 0.5 * off
        y = cc + rng.uniform(-0.25, 0.25, size=(7, 3))
        q = rng.uniform(-1, 1, 7)
        Mp_direct += O.p2m(p, cp, y, q)
        Mp_chain += O.m2m(p, O.p2m(p, cc, y, q), cc - cp)
    assert np.max(np.abs(Mp_chain - Mp_direct)) <= 1e-13 * np.max(np.abs(Mp_direct))


def test_m2m_monopole_shift_is_point_charge(O):
    M = np.zeros(O.nterms(10), complex)
    M[0] = 1.5
    b = np.array([0.1, -0.2, 0.05])
    Mp = O.m2m(10, M, b)
    x = np.array([[3.0, 2.0, -1.0]])
    phi, _ = O.m2p(10, Mp, np.zeros(3), x)
    assert phi[0] == pytest.approx(1.5 / np.linalg.norm(x[0] - b), rel=1e-10)


def test_l2l_identity_constant_and_exact_chain(O):
    p = 10
    L = rng.normal(size=O.nterms(p)) + 1j * rng.normal(size=O.nterms(p))
    # make it the local expansion of a real field: L_n^{-m} = (-1)^m conj(L_n^m)
    for n in range(p + 1):
        L[O.idx(n, 0)] = L[O.idx(n, 0)].real
        for m in range(1, n + 1):
            L[O.idx(n, -m)] = (-1) ** m * np.conj(L[O.idx(n, m)])
    np.testing.assert_allclose(O.l2l(p, L, [0, 0, 0]), L, atol=1e-14)
    Lc = np.zeros_like(L)
    Lc[0] = 0.7
    np.testing.assert_allclose(O.l2l(p, Lc, [0.3, -0.1, 0.2]), Lc, atol=1e-15)
    # L2L then L2P == L2P (exact; polynomial re-expansion)
    cp = np.zeros(3)
    e = np.array([0.25, -0.25, 0.25])
    x = e + rng.uniform(-0.2, 0.2, size=(6, 3))
    phi0, g0 = O.l2p(p, L, cp, x)
    phi1, g1 = O.l2p(p, O.l2l(p, L, e), e, x)
    np.testing.assert_allclose(phi1, phi0, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(g1, g0, rtol=1e-11, atol=1e-11)


def test_l2p_constant_term(O):
    L = np.zeros(O.nterms(5), complex)
    L[0] = 4.0  # potential += c, force += 0
    phi, grad = O.l2p(5, L, np.zeros(3), rng.normal(size=(4, 3)))
    np.testing.assert_allclose(phi, 4.0)
    assert np.all(grad == 0)


# ---------------- M2L ----------------
def test_m2l_monopole_gives_q_over_R(O):
    # monopole source, local expansion evaluated at the target centre gives q/R.
    M = np.zeros(O.nterms(10), complex)
    M[0] = 2.0
    d = np.array([2.0, -1.0, 1.5])
    L = O.m2l(10, M, d)
    phi, grad = O.l2p(10, L, np.zeros(3), np.zeros((1, 3)))
    assert phi[0] == pytest.approx(2.0 / np.linalg.norm(d), rel=1e-14)
    np.testing.assert_allclose(grad[0], -2.0 * d / np.linalg.norm(d) ** 3, rtol=1e-12)


def _m2l_case(O, p, theta_pair, seed=7):
    rng = np.random.default_rng(seed)
    cs = np.zeros(3)
    rs = 0.5
    y = cs + rng.uniform(-rs, rs, size=(30, 3))
    q = rng.uniform(0.1, 1.0, 30)
    R = 2 * rs / theta_pair
    ct = cs + R * np.array([0.6, 0.64, 0.48])
    x = ct + rng.uniform(-rs, rs, size=(30, 3))
    L = O.m2l(p, O.p2m(p, cs, y, q), ct - cs)
    phi, grad = O.l2p(p, L, ct, x)
    pd, gd = O.p2p(x, y, q)
    return O.rel_l2(phi, pd), O.rel_l2(grad, gd)


def test_m2l_l2p_matches_direct(O):
    # theta_pair = 0.3, p=10 -> <= 1e-5 relative
    ep, eg = _m2l_case(O, 10, 0.3)
    assert ep < 1e-5 and eg < 1e-4


def test_m2l_converges_in_p(O):
    errs = [_m2l_case(O, p, 0.4)[0] for p in (2, 4, 6, 8, 10, 12)]
    assert all(b < a for a, b in zip(errs, errs[1:])), errs


def test_m2p_equals_l2p_of_m2l(O):
    # M2P ~= L2P(M2L) on well-separated pairs, to truncation order.
    p = 12
    y = rng.uniform(-0.5, 0.5, size=(10, 3))
    q = rng.uniform(-1, 1, 10)
    M = O.p2m(p, np.zeros(3), y, q)
    ct = np.array([3.0, 2.0, 1.0])
    x = ct + rng.uniform(-0.5, 0.5, size=(8, 3))
    a, ga = O.m2p(p, M, np.zeros(3), x)
    b, gb = O.l2p(p, O.m2l(p, M, ct), ct, x)
    assert O.rel_l2(b, a) < 1e-6 and O.rel_l2(gb, ga) < 1e-5


# ---------------- gradients by finite differences ----------------
@pytest.mark.parametrize("which", ["m2p", "l2p"])
def test_gradient_matches_finite_difference(O, which):
    p = 8
    y = rng.uniform(-0.5, 0.5, size=(10, 3))
    q = rng.uniform(-1, 1, 10)
    M = O.p2m(p, np.zeros(3), y, q)
    if which == "m2p":
        fn = lambda x: O.m2p(p, M, np.zeros(3), x)
        x0 = np.array([[2.0, 1.5, -1.0]])
    else:
        ct = np.array([3.0, 2.0, 1.0])
        L = O.m2l(p, M, ct)
        fn = lambda x: O.l2p(p, L, ct, x)
        x0 = ct + np.array([[0.2, -0.1, 0.15]])
    _, g = fn(x0)
    h = 1e-5
    fd = np.zeros(3)
    for a in range(3):
        e = np.zeros((1, 3))
        e[0, a] = h
        fd[a] = (fn(x0 + e)[0][0] - fn(x0 - e)[0][0]) / (2 * h)
    np.testing.assert_allclose(g[0], fd, rtol=1e-6, atol=1e-9)


# ---------------- P2P ----------------
def test_p2p_self_exclusion_and_momentum(O):
    y = rng.uniform(size=(40, 3))
    q = rng.uniform(-1, 1, 40)
    phi, grad = O.p2p(y, y, q)
    p1, g1 = O.p2p(y[:1], y[:1], q[:1])
    assert p1[0] == 0 and np.all(g1 == 0)
    # sum_i q_i f_i = 0 by pairwise antisymmetry
    mom = (q[:, None] * grad).sum(axis=0)
    assert np.max(np.abs(mom)) < 1e-12 * np.max(np.abs(q[:, None] * grad))
