"""Oracle pins: the whole method against the exact direct sum.

PAPER.md:47 — p=10 gives 4 significant digits in the potential (north_star gate: 1e-4 relative
L2 vs direct); PAPER.md:174 — p=8 FMM gives 4 digits in the force (gated at 1e-3, S:517 margin);
error falls monotonically in p; closed-form golden charges (tests/golden/*.json).
"""
import json
import os

import numpy as np
import pytest

from fmm_inputs import make_particles

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("name", ["two_charges", "three_charges"])
@pytest.mark.parametrize("mode", ["DIRECT", "FMM", "HYBRID"])
def test_golden_charges(O, name, mode):
    g = json.load(open(os.path.join(GOLD, name + ".json")))
    xyz = np.array(g["xyz"], np.float32)
    q = np.array(g["q"], np.float32)
    res = O.fmm(xyz, q, 4, 0.5, 1, getattr(O, mode), cost=(1e-9, 1e-7, 1e-5))
    np.testing.assert_allclose(res.phi, g["phi"], rtol=1e-12)
    np.testing.assert_allclose(res.grad, g["grad"], rtol=1e-12, atol=1e-15)
    d = O.direct(xyz, q)
    np.testing.assert_allclose(d[0], g["phi"], rtol=1e-15)
    np.testing.assert_allclose(d[1], g["grad"], rtol=1e-15, atol=1e-16)


def test_convergence_ladder_c1(O):
    # C1: N=1000 uniform, theta=0.5, ncrit=16; error vs direct falls monotonically in p.
    xyz, q = make_particles(1000, "uniform", 1)
    d = O.direct(xyz, q)
    ep, eg = [], []
    for p in (2, 4, 6, 8, 10, 12):
        r = O.fmm(xyz, q, p, 0.5, 16, O.FMM, want_structure=False)
        ep.append(O.rel_l2(r.phi, d[0]))
        eg.append(O.rel_l2(r.grad, d[1]))
    assert all(b < a for a, b in zip(ep, ep[1:])), ep
    assert all(b < a for a, b in zip(eg, eg[1:])), eg
    assert ep[4] < 1e-4  # p=10: 4 digits in the potential
    assert eg[3] < 1e-3  # p=8: 4 digits in the force, one-decade margin


@pytest.mark.parametrize("dist,theta", [("uniform", 0.4), ("uniform", 0.5), ("plummer", 0.4),
                                        ("mixed", 0.5), ("shell", 0.5)])
@pytest.mark.parametrize("mode", ["FMM", "TREECODE", "HYBRID"])
def test_p10_meets_four_digits(O, dist, theta, mode):
    xyz, q = make_particles(4000, dist, 3)
    d = O.direct(xyz, q)
    r = O.fmm(xyz, q, 10, theta, 32, getattr(O, mode), cost=(2e-11, 3e-9, 5e-7), want_structure=False)
    assert O.rel_l2(r.phi, d[0]) < 1e-4
    assert O.rel_l2(r.grad, d[1]) < 1e-3


def test_sampled_mode_equals_full(O):
    xyz, q = make_particles(6000, "plummer", 8)
    s = np.random.default_rng(0).choice(len(q), 64, replace=False)
    for mode in (O.FMM, O.HYBRID, O.TREECODE):
        full = O.fmm(xyz, q, 6, 0.45, 24, mode, cost=(2e-11, 3e-9, 5e-7), want_structure=False)
        smp = O.fmm(xyz, q, 6, 0.45, 24, mode, cost=(2e-11, 3e-9, 5e-7), sample=s)
        np.testing.assert_allclose(smp.phi, full.phi[s], rtol=1e-12)
        np.testing.assert_allclose(smp.grad, full.grad[s], rtol=1e-10, atol=1e-14)


def test_dyadic_translation_invariance(O):
    # S:230 restricted to shifts that keep the keys (coordinates on a 2^-12 grid, shift by 1).
    rng = np.random.default_rng(3)
    xyz = (rng.integers(0, 4096, size=(2000, 3)) / 4096.0).astype(np.float32)
    q = rng.uniform(-1, 1, 2000).astype(np.float32)
    a = O.fmm(xyz, q, 8, 0.5, 20, O.FMM)
    b = O.fmm(xyz + np.float32(1.0), q, 8, 0.5, 20, O.FMM)
    assert np.array_equal(a.sorted_keys, b.sorted_keys)
    assert O.rel_l2(b.phi, a.phi) < 1e-12 and O.rel_l2(b.grad, a.grad) < 1e-10


def test_degenerate_inputs(O):
    r = O.fmm(np.zeros((0, 3), np.float32), np.zeros(0, np.float32), 4, 0.5, 8)
    assert r.phi.size == 0
    # coincident distinct particles contribute nothing to each other (DESIGN reading R13)
    xyz = np.array([[0.2, 0.2, 0.2], [0.2, 0.2, 0.2], [0.7, 0.2, 0.2]], np.float32)
    q = np.ones(3, np.float32)
    d = O.direct(xyz, q)
    np.testing.assert_allclose(O.fmm(xyz, q, 4, 0.5, 1, O.DIRECT).phi, d[0], rtol=1e-14)
    np.testing.assert_allclose(O.fmm(xyz, q, 4, 0.5, 2, O.FMM).phi, d[0], rtol=1e-14)  # all near field
    np.testing.assert_allclose(O.fmm(xyz, q, 16, 0.5, 1, O.FMM).phi, d[0], rtol=1e-4)
    assert d[0][0] == pytest.approx(2.0, rel=1e-6)  # only the particle at distance 0.5
    # all particles at one point: tree depth capped at level 21
    xyz = np.full((40, 3), 0.3, np.float32)
    r = O.fmm(xyz, np.ones(40, np.float32), 3, 0.5, 4, O.FMM)
    assert r.tree["level"].max() == 21 and np.all(r.phi == 0)
