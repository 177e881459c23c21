"""Oracle pins: MAC, kind selection and the LIFO dual traversal.

Pinned by closed-form near-pair counts on full uniform octrees (PAPER.md:168 'theta=0.5 is
equivalent to a 3x3x3 neighbor list'; tests/golden/near_pair_counts.json), exact pair coverage
(every ordered particle pair covered by exactly one task), selector forcing and the
S:338-345 cost examples.
"""
import json
import os

import numpy as np
import pytest

from fmm_inputs import make_particles

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def full_grid(L):
    """One particle at the centre of each of the 8^L finest cells of [0,1)^3."""
    g = (np.arange(2 ** L) + 0.5) / 2 ** L
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    xyz = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1).astype(np.float32)
    return xyz, np.full(len(xyz), 1.0 / len(xyz), np.float32)


@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLD, "near_pair_counts.json")))["cases"],
                         ids=lambda c: f"L{c['L']}-t{c['theta']}")
def test_near_pair_closed_form(O, case):
    xyz, q = full_grid(case["L"])
    res = O.fmm(xyz, q, 1, case["theta"], 1, O.FMM)
    lev = res.tree["level"]
    assert lev.max() == case["L"] and np.sum(lev == case["L"]) == 8 ** case["L"]
    kinds = res.tasks["kind"]
    assert np.sum(kinds == O.K_P2P) == case["near"]
    assert np.sum(kinds == O.K_M2P) == 0


def test_strict_mac_mutation_golden(O):
    """The golden's strict-MAC count (SPEC S:257 '<' instead of the '<=' reading R5): accept-if-<
    at theta = 0.5 equals accept-if-<= at theta just below 0.5 on this exact geometry (no pair has
    (r_t + r_s) / R strictly between the two). It must give the extra face second-neighbour pairs
    6 (2^L - 2) 4^L = 21,504 at L = 4, i.e. 118,840, and differ from the closed form we pin."""
    g = json.load(open(os.path.join(GOLD, "near_pair_counts.json")))
    mut = g["strict_mutation"]
    base = [c for c in g["cases"] if c["L"] == mut["L"] and c["theta"] == mut["theta"]][0]
    L = mut["L"]
    assert mut["near"] == base["near"] + 6 * (2 ** L - 2) * 4 ** L
    xyz, q = full_grid(L)
    res = O.fmm(xyz, q, 1, mut["theta"] * (1 - 1e-12), 1, O.FMM)
    assert np.sum(res.tasks["kind"] == O.K_P2P) == mut["near"] != base["near"]


def coverage(O, res, n):
    cov = np.zeros((n, n), np.int32)
    for kind, tb, tc, sb, sc in O.task_ranges(res):
        cov[tb:tb + tc, sb:sb + sc] += 1
    return cov


@pytest.mark.parametrize("mode", ["FMM", "TREECODE", "HYBRID"])
@pytest.mark.parametrize("dist", ["uniform", "shell", "plummer"])
@pytest.mark.parametrize("ncrit", [1, 20, 50, 200])
def test_exact_pair_coverage(O, mode, dist, ncrit):
    # every ordered (target, source) particle pair is covered by exactly one task.
    for seed in (1, 2, 3):
        xyz, q = make_particles(400, dist, seed)
        cost = np.random.default_rng(seed).uniform(1e-9, 1e-6, 3)
        res = O.fmm(xyz, q, 2, 0.5, ncrit, getattr(O, mode), cost=cost)
        cov = coverage(O, res, len(q))
        assert np.all(cov == 1), (mode, dist, ncrit, seed)


def test_selector_forcing(O):
    xyz, q = make_particles(1500, "plummer", 4)
    fmm = O.fmm(xyz, q, 6, 0.5, 16, O.FMM)
    hyb0 = O.fmm(xyz, q, 6, 0.5, 16, O.HYBRID, cost=(1e-9, 1e-7, 0.0))  # t_ml = 0 -> always M2L
    a, b = O.canonical_tasks(fmm.tasks), O.canonical_tasks(hyb0.tasks)
    assert np.array_equal(a, b)
    tre = O.fmm(xyz, q, 6, 0.5, 16, O.TREECODE)
    assert np.all(tre.tasks["kind"] != O.K_M2L)
    # t_pp = 0 -> every accepted pair is P2P -> the result is the direct sum
    hp = O.fmm(xyz, q, 6, 0.5, 16, O.HYBRID, cost=(0.0, 1e-7, 1e-5))
    assert np.all(hp.tasks["kind"] == O.K_P2P)
    d = O.direct(xyz, q)
    assert O.rel_l2(hp.phi, d[0]) < 1e-12 and O.rel_l2(hp.grad, d[1]) < 1e-12


def test_cost_model_examples(O):
    # S:338-345 with exactly representable per-unit times (powers of two) so the tie is exact.
    cost = (2.0 ** -30, 2.0 ** -24, 2.0 ** -16)  # n_t = n_s = 2^7: P2P 2^-16, M2P 2^-17, M2L 2^-16
    assert O.select_kind(O.HYBRID, cost, 128, 128) == O.K_M2P
    cost = (2.0 ** -30, 2.0 ** -23, 2.0 ** -16)  # n=128: P2P = M2P = M2L = 2^-16 -> tie -> M2L
    assert O.select_kind(O.HYBRID, cost, 128, 128) == O.K_M2L
    cost = (1e-9, 1e-7, 1e-5)
    assert O.select_kind(O.HYBRID, cost, 10, 10) == O.K_P2P
    assert O.select_kind(O.HYBRID, cost, 1000, 1000) == O.K_M2L
    # scale invariance on exactly scaled costs
    for nt, ns in [(3, 5), (50, 70), (1, 1000), (900, 2)]:
        k = O.select_kind(O.HYBRID, cost, nt, ns)
        assert O.select_kind(O.HYBRID, [c * 4.0 for c in cost], nt, ns) == k
    assert O.select_kind(O.FMM, cost, 1, 1) == O.K_M2L
    assert O.select_kind(O.TREECODE, cost, 1, 1) == O.K_M2P


def test_single_leaf_tree_single_p2p(O):
    xyz, q = make_particles(10, "uniform", 3)
    res = O.fmm(xyz, q, 4, 0.5, 16, O.FMM)  # two single-leaf trees -> one P2P
    assert len(res.tasks["kind"]) == 1 and res.tasks["kind"][0] == O.K_P2P


def test_theta_monotonicity(O):
    xyz, q = make_particles(3000, "uniform", 5)
    d = O.direct(xyz, q)
    errs = [O.rel_l2(O.fmm(xyz, q, 4, th, 16, O.FMM, want_structure=False).phi, d[0])
            for th in (0.7, 0.5, 0.35, 0.25)]
    assert all(b < a for a, b in zip(errs, errs[1:])), errs


def test_coverage_check_detects_mutations(O):
    # SURVEY §4.2 mutation test: the exact-coverage check must fail when the task set is wrong --
    # a dropped task leaves pairs uncovered, a duplicated task covers pairs twice
    xyz, q = make_particles(300, "uniform", 9)
    res = O.fmm(xyz, q, 2, 0.5, 16, O.HYBRID, cost=(2e-12, 6e-11, 2.5e-9))
    assert np.all(coverage(O, res, len(q)) == 1)
    t = res.tasks
    for mutate in ("drop", "dup"):
        idx = np.arange(len(t["kind"]))
        idx = idx[1:] if mutate == "drop" else np.concatenate([idx, idx[:1]])
        res.tasks = {k: np.asarray(v)[idx] for k, v in t.items()}
        assert not np.all(coverage(O, res, len(q)) == 1), mutate
    res.tasks = t


def test_work_count_scaling(O):
    # the FMM is O(N) (cell-cell interactions per particle constant), the treecode
    # O(N log N) (cell-particle evaluations per particle grow with log N). Counts from the
    # oracle's lists on uniform cubes at a fixed occupancy (ncrit) over a 64x range of N.
    Ns = [2000, 16000, 128000]
    fmm_work, tree_work = [], []
    for n in Ns:
        xyz, q = make_particles(n, "uniform", 11)
        r = O.fmm(xyz, q, 1, 0.5, 16, O.FMM)
        fmm_work.append(np.sum(r.tasks["kind"] == O.K_M2L))
        r = O.fmm(xyz, q, 1, 0.5, 16, O.TREECODE)
        rng = O.task_ranges(r)
        tree_work.append(int(np.sum(rng[rng[:, 0] == O.K_M2P, 2])))  # target particles x cells
    s_fmm = np.polyfit(np.log(Ns), np.log(fmm_work), 1)[0]
    s_tree = np.polyfit(np.log(Ns), np.log(tree_work), 1)[0]
    # per-particle work: the FMM's converges to a constant (its growth at these sizes is the
    # shrinking share of boundary cells, and its increments per 8x in N shrink); the treecode's
    # grows like log N (increments per 8x in N do not shrink)
    f_pp = np.array(fmm_work) / np.array(Ns)
    t_pp = np.array(tree_work) / np.array(Ns)
    df, dt = np.diff(f_pp), np.diff(t_pp)
    assert df[1] < 0.8 * df[0], f_pp
    assert dt[1] > 0.9 * dt[0], t_pp
    assert s_tree > s_fmm + 0.15, (s_tree, s_fmm)
    assert 0.9 < s_fmm < 1.2 and s_tree < 1.5, (s_fmm, s_tree)
