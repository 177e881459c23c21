"""Oracle pins: root cube, Morton keys, adaptive octree.

Pinned against a brute-force *geometric* octree (recursive cube subdivision by coordinate
comparison, no bit interleaving), the S:102-103 examples and the S:116-120 invariants.
"""
import math

import numpy as np
import pytest

from fmm_inputs import make_particles


def naive_octree(xyz, ncrit):
    """Recursive geometric subdivision of the power-of-two root cube (c2, c3)."""
    x = xyz.astype(np.float64)
    mn, mx = x.min(0), x.max(0)
    ext = float((mx - mn).max())
    L = 1.0 if ext == 0 else 2.0 ** math.ceil(math.log2(ext))
    origin = 0.5 * (mn + mx) - 0.5 * L
    cells = []

    def rec(idx, lo, w, level):
        cells.append((level, frozenset(idx.tolist())))
        if len(idx) <= ncrit or level >= 21:
            return
        c = lo + 0.5 * w
        for o in range(8):
            bits = [(o >> 2) & 1, (o >> 1) & 1, o & 1]
            sel = np.ones(len(idx), bool)
            for a in range(3):
                sel &= (x[idx, a] >= c[a]) if bits[a] else (x[idx, a] < c[a])
            if sel.any():
                rec(idx[sel], lo + 0.5 * w * np.array(bits), 0.5 * w, level + 1)

    rec(np.arange(len(x)), origin, L, 0)
    return sorted(cells, key=lambda c: (c[0], min(c[1]))), origin, L


def oracle_cells(res):
    t = res.tree
    return sorted(((int(l), frozenset(res.perm[b:b + c].tolist()))
                   for l, b, c in zip(t["level"], t["begin"], t["count"])), key=lambda c: (c[0], min(c[1])))


@pytest.mark.parametrize("dist,n,ncrit,seed", [("uniform", 64, 1, 1), ("uniform", 300, 8, 2),
                                               ("plummer", 200, 4, 3), ("shell", 150, 5, 4),
                                               ("mixed", 100, 2, 5)])
def test_tree_matches_geometric_octree(O, dist, n, ncrit, seed):
    xyz, q = make_particles(n, dist, seed)
    res = O.fmm(xyz, q, 2, 0.5, ncrit, O.FMM)
    naive, origin, L = naive_octree(xyz, ncrit)
    assert res.L == L and np.allclose(res.origin, origin, rtol=0, atol=0)
    assert oracle_cells(res) == naive


def test_eight_octant_particles(O):
    # 8 particles at (+-.5,+-.5,+-.5), ncrit=1 -> 9 cells, 8 leaves; x bit is the MSB.
    pts = np.array([[sx, sy, sz] for sx in (-.5, .5) for sy in (-.5, .5) for sz in (-.5, .5)], np.float32)
    res = O.fmm(pts, np.ones(8, np.float32), 2, 0.5, 1, O.FMM)
    t = res.tree
    assert len(t["level"]) == 9 and np.sum(t["level"] == 1) == 8
    assert list(t["prefix"][t["level"] == 1]) == list(range(8))
    np.testing.assert_array_equal(res.perm, np.arange(8))  # generated in octant order already


def test_single_particle_single_leaf(O):
    res = O.fmm(np.array([[0.3, 0.2, 0.1]], np.float32), np.ones(1, np.float32), 3, 0.5, 4, O.FMM)
    assert len(res.tree["level"]) == 1 and res.phi[0] == 0.0


def test_root_cube_and_key_containment(O):
    xyz, _ = make_particles(5000, "plummer", 9)
    o, L, keys = O.morton_keys(xyz)
    ext = float((xyz.max(0).astype(np.float64) - xyz.min(0)).max())
    assert L >= ext and L / 2 < ext and math.log2(L) == int(math.log2(L))
    # each particle lies in the finest cube its key names (decode by bit comparison)
    g = np.zeros((len(keys), 3), np.int64)
    for b in range(21):
        for a in range(3):
            g[:, a] |= ((keys >> np.uint64(3 * b + 2 - a)) & np.uint64(1)).astype(np.int64) << b
    w = L / 2 ** 21
    lo = o + g * w
    x = xyz.astype(np.float64)
    inside = (x >= lo) & (x < lo + w)
    at_top = (g == 2 ** 21 - 1) & (x >= lo)  # the clamped upper face
    assert np.all(inside | at_top)


def test_tree_invariants(O):
    xyz, q = make_particles(3000, "plummer", 11)
    depths = []
    for ncrit in (4, 16, 64, 256):
        res = O.fmm(xyz, q, 2, 0.5, ncrit, O.FMM)
        t = res.tree
        lev, pre, beg, cnt = t["level"], t["prefix"], t["begin"], t["count"]
        cells = {(int(l), int(p)): (int(b), int(c)) for l, p, b, c in zip(lev, pre, beg, cnt)}
        leaves = []
        for (l, p), (b, c) in cells.items():
            kids = [cells[(l + 1, p * 8 + o)] for o in range(8) if (l + 1, p * 8 + o) in cells]
            if kids:
                assert c > ncrit  # split only when count > ncrit
                assert sum(k[1] for k in kids) == c  # containment / partition of the parent
                assert min(k[0] for k in kids) == b
            else:
                assert c <= ncrit or l == 21
                leaves.append((b, c))
            if l > 0:
                assert (l - 1, p // 8) in cells
        leaves.sort()
        assert leaves[0][0] == 0 and sum(c for _, c in leaves) == len(q)
        assert all(b0 + c0 == b1 for (b0, c0), (b1, _) in zip(leaves, leaves[1:]))
        depths.append(int(lev.max()))
    assert depths == sorted(depths, reverse=True)  # depth monotone in ncrit


def test_sort_is_stable_by_key_then_index(O):
    xyz = np.array([[0.5, 0.5, 0.5]] * 3 + [[0.1, 0.1, 0.1]] * 2, np.float32)
    o, L, keys = O.morton_keys(xyz)
    res = O.fmm(xyz, np.ones(5, np.float32), 2, 0.5, 1, O.FMM)
    assert list(res.perm) == [3, 4, 0, 1, 2]


def test_nonfinite_input_rejected(O):
    xyz, q = make_particles(10, "uniform", 1)
    xyz[3, 1] = np.nan
    with pytest.raises(ValueError):
        O.fmm(xyz, q, 2, 0.5, 4)
