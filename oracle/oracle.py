"""ctypes front-end of the FP64 CPU oracle (oracle/*.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, by __graft_entry__.smoke() (to check the GPU
result) and by bench.py's cpu_baseline / `--impl reference` legs. The product path
(paper_1108_5815_b200) never imports this module, and this module never imports the product.
Each function names the PAPER.md / SPEC.md passage it follows in the C source it wraps.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SOURCES = ["harmonics.c", "cartesian.c", "tree.c", "traversal.c", "evaluate.c"]

HYBRID, FMM, TREECODE, DIRECT = 0, 1, 2, 3
K_M2L, K_M2P, K_P2P = 0, 1, 2
KIND_NAMES = {K_M2L: "M2L", K_M2P: "M2P", K_P2P: "P2P"}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (FP64, no FP contraction so the MAC is bit-reproducible)."""
    srcs = [os.path.join(HERE, s) for s in SOURCES] + [os.path.join(HERE, "oracle.h")]
    if not force and os.path.exists(LIB_PATH):
        if os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(s) for s in srcs):
            return LIB_PATH
    cmd = ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-fcx-limited-range", "-o", LIB_PATH + ".tmp"] + [os.path.join(HERE, s) for s in SOURCES] + ["-lm"]
    subprocess.check_call(cmd)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        dp, fp, i64p, u64p, i32p = (C.POINTER(C.c_double), C.POINTER(C.c_float),
                                    C.POINTER(C.c_int64), C.POINTER(C.c_uint64), C.POINTER(C.c_int32))
        L.orc_harm_R.argtypes = [dp, C.c_int, dp]
        L.orc_harm_I.argtypes = [dp, C.c_int, dp]
        L.orc_p2m.argtypes = [C.c_int, dp, C.c_int64, dp, dp, dp]
        L.orc_m2m.argtypes = [C.c_int, dp, dp, dp]
        L.orc_m2l.argtypes = [C.c_int, dp, dp, dp]
        L.orc_l2l.argtypes = [C.c_int, dp, dp, dp]
        L.orc_l2p.argtypes = [C.c_int, dp, dp, C.c_int64, dp, dp, dp]
        L.orc_m2p.argtypes = [C.c_int, dp, dp, C.c_int64, dp, dp, dp]
        L.orc_p2p.argtypes = [C.c_int64, dp, C.c_int64, dp, dp, dp, dp]
        L.orc_root_cube.argtypes = [fp, C.c_int64, dp, dp]
        L.orc_root_cube.restype = C.c_int
        L.orc_morton_keys.argtypes = [fp, C.c_int64, dp, C.c_double, u64p]
        L.orc_fmm_run.argtypes = [fp, fp, C.c_int64, C.c_int, C.c_double, C.c_int, C.c_int, dp,
                                  i64p, C.c_int64, dp, dp, dp]
        L.orc_fmm_run.restype = C.c_void_p
        L.orc_fmm_run_basis.argtypes = L.orc_fmm_run.argtypes + [C.c_int]
        L.orc_fmm_run_basis.restype = C.c_void_p
        L.orc_cart_count.argtypes = [C.c_int]
        L.orc_cart_count.restype = C.c_int
        L.orc_cart_index.argtypes = [C.c_int, C.c_int, C.c_int]
        L.orc_cart_index.restype = C.c_int
        L.orc_cart_multi.argtypes = [C.c_int, C.POINTER(C.c_int)]
        L.orc_cart_derivs.argtypes = [dp, C.c_int, dp]
        L.orc_cart_p2m.argtypes = [C.c_int, dp, C.c_int64, dp, dp, dp]
        L.orc_cart_m2m.argtypes = [C.c_int, dp, dp, dp]
        L.orc_cart_m2l.argtypes = [C.c_int, dp, dp, dp]
        L.orc_cart_l2l.argtypes = [C.c_int, dp, dp, dp]
        L.orc_cart_l2p.argtypes = [C.c_int, dp, dp, C.c_int64, dp, dp, dp]
        L.orc_cart_m2p.argtypes = [C.c_int, dp, dp, C.c_int64, dp, dp, dp]
        L.orc_fmm_ncells.argtypes = [C.c_void_p]
        L.orc_fmm_ncells.restype = C.c_int64
        L.orc_fmm_ntasks.argtypes = [C.c_void_p]
        L.orc_fmm_ntasks.restype = C.c_int64
        L.orc_fmm_tree.argtypes = [C.c_void_p, i32p, u64p, i64p, i64p]
        L.orc_fmm_tasks.argtypes = [C.c_void_p, i32p, i32p, u64p, i32p, u64p]
        L.orc_fmm_perm.argtypes = [C.c_void_p, i64p, u64p]
        L.orc_fmm_root.argtypes = [C.c_void_p, dp, dp]
        L.orc_fmm_free.argtypes = [C.c_void_p]
        L.orc_direct.argtypes = [fp, fp, C.c_int64, i64p, C.c_int64, dp, dp]
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _cx(a):  # complex128 array -> double*
    return a.view(np.float64).ctypes.data_as(C.POINTER(C.c_double))


def nterms(p: int) -> int:
    return (p + 1) * (p + 1)


def idx(n: int, m: int) -> int:
    return n * n + n + m


# ---------------- harmonics and operators ----------------
def harm_R(x, P):
    out = np.zeros(nterms(P), np.complex128)
    lib().orc_harm_R(_p(np.ascontiguousarray(x, np.float64), C.c_double), P, _cx(out))
    return out


def harm_I(x, P):
    out = np.zeros(nterms(P), np.complex128)
    lib().orc_harm_I(_p(np.ascontiguousarray(x, np.float64), C.c_double), P, _cx(out))
    return out


def p2m(p, c, y, q):
    M = np.zeros(nterms(p), np.complex128)
    y = np.ascontiguousarray(y, np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(q, np.float64)
    lib().orc_p2m(p, _p(np.ascontiguousarray(c, np.float64), C.c_double), len(q),
                  _p(y, C.c_double), _p(q, C.c_double), _cx(M))
    return M


def _shift(fn, p, X, v):
    out = np.zeros(nterms(p), np.complex128)
    X = np.ascontiguousarray(X, np.complex128)
    fn(p, _cx(X), _p(np.ascontiguousarray(v, np.float64), C.c_double), _cx(out))
    return out


def m2m(p, Mc, b):
    return _shift(lib().orc_m2m, p, Mc, b)


def m2l(p, Ms, d):
    return _shift(lib().orc_m2l, p, Ms, d)


def l2l(p, Lp, e):
    return _shift(lib().orc_l2l, p, Lp, e)


def _eval(fn, p, X, c, x):
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    phi = np.zeros(len(x))
    grad = np.zeros((len(x), 3))
    fn(p, _cx(np.ascontiguousarray(X, np.complex128)),
       _p(np.ascontiguousarray(c, np.float64), C.c_double), len(x), _p(x, C.c_double),
       _p(phi, C.c_double), _p(grad, C.c_double))
    return phi, grad


def l2p(p, L, c, x):
    return _eval(lib().orc_l2p, p, L, c, x)


def m2p(p, M, c, x):
    return _eval(lib().orc_m2p, p, M, c, x)


def p2p(xt, ys, qs):
    xt = np.ascontiguousarray(xt, np.float64).reshape(-1, 3)
    ys = np.ascontiguousarray(ys, np.float64).reshape(-1, 3)
    qs = np.ascontiguousarray(qs, np.float64)
    phi = np.zeros(len(xt))
    grad = np.zeros((len(xt), 3))
    lib().orc_p2p(len(xt), _p(xt, C.c_double), len(ys), _p(ys, C.c_double), _p(qs, C.c_double),
                  _p(phi, C.c_double), _p(grad, C.c_double))
    return phi, grad


# ---------------- keys ----------------
# ---- Cartesian Taylor operators (cartesian.c; NEXT-2) --------------------------------------
def cart_count(p: int) -> int:
    return int(lib().orc_cart_count(p))


def cart_index(kx, ky, kz) -> int:
    return int(lib().orc_cart_index(kx, ky, kz))


def cart_multi(p):
    k3 = np.zeros((cart_count(p), 3), np.int32)
    lib().orc_cart_multi(p, _p(k3, C.c_int))
    return k3


def cart_derivs(d, P):
    a = np.zeros(cart_count(P))
    lib().orc_cart_derivs(_p(np.ascontiguousarray(d, np.float64), C.c_double), P, _p(a, C.c_double))
    return a


def cart_p2m(p, c, y, q):
    y = np.ascontiguousarray(y, np.float64).reshape(-1, 3)
    M = np.zeros(cart_count(p))
    lib().orc_cart_p2m(p, _p(np.ascontiguousarray(c, np.float64), C.c_double), len(y),
                       _p(y, C.c_double), _p(np.ascontiguousarray(q, np.float64), C.c_double),
                       _p(M, C.c_double))
    return M


def _cart_shift(fn, p, X, v):
    out = np.zeros(cart_count(p))
    fn(p, _p(np.ascontiguousarray(X, np.float64), C.c_double),
       _p(np.ascontiguousarray(v, np.float64), C.c_double), _p(out, C.c_double))
    return out


def cart_m2m(p, Mc, b):
    return _cart_shift(lib().orc_cart_m2m, p, Mc, b)


def cart_m2l(p, Ms, d):
    return _cart_shift(lib().orc_cart_m2l, p, Ms, d)


def cart_l2l(p, Lp, e):
    return _cart_shift(lib().orc_cart_l2l, p, Lp, e)


def _cart_eval(fn, p, X, c, x):
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    phi = np.zeros(len(x))
    grad = np.zeros((len(x), 3))
    fn(p, _p(np.ascontiguousarray(X, np.float64), C.c_double),
       _p(np.ascontiguousarray(c, np.float64), C.c_double), len(x), _p(x, C.c_double),
       _p(phi, C.c_double), _p(grad, C.c_double))
    return phi, grad


def cart_l2p(p, L, c, x):
    return _cart_eval(lib().orc_cart_l2p, p, L, c, x)


def cart_m2p(p, M, c, x):
    return _cart_eval(lib().orc_cart_m2p, p, M, c, x)


def root_cube(xyz):
    xyz = np.ascontiguousarray(xyz, np.float32)
    o = np.zeros(3)
    L = np.zeros(1)
    rc = lib().orc_root_cube(_p(xyz, C.c_float), len(xyz), _p(o, C.c_double), _p(L, C.c_double))
    if rc != 0:
        raise ValueError("non-finite coordinates")
    return o, float(L[0])


def morton_keys(xyz):
    xyz = np.ascontiguousarray(xyz, np.float32)
    o, L = root_cube(xyz)
    keys = np.zeros(len(xyz), np.uint64)
    lib().orc_morton_keys(_p(xyz, C.c_float), len(xyz), _p(o, C.c_double), L, _p(keys, C.c_uint64))
    return o, L, keys


# ---------------- whole method ----------------
@dataclass
class OracleResult:
    phi: np.ndarray
    grad: np.ndarray
    phases: np.ndarray  # seconds: build, upward, traverse, evaluate, downward
    tree: dict
    tasks: dict
    perm: np.ndarray
    sorted_keys: np.ndarray
    origin: np.ndarray
    L: float


def fmm(xyz, q, p, theta, ncrit, mode=HYBRID, cost=(1.0, 1.0, 1.0), sample=None,
        want_structure=True, basis="spherical") -> OracleResult:
    """The whole method in FP64. cost = (t_pp, t_mp, t_ml) seconds per unit;
    basis = "spherical" (harmonics.c) or "cartesian" (cartesian.c, NEXT-2)."""
    xyz = np.ascontiguousarray(xyz, np.float32).reshape(-1, 3)
    q = np.ascontiguousarray(q, np.float32)
    n = len(q)
    cost_a = np.ascontiguousarray(cost, np.float64)
    if sample is not None:
        sample = np.ascontiguousarray(sample, np.int64)
        nout = len(sample)
        sp = _p(sample, C.c_int64)
    else:
        nout, sp = n, None
    phi = np.zeros(nout)
    grad = np.zeros((nout, 3))
    phases = np.zeros(5)
    L = lib()
    h = L.orc_fmm_run_basis(_p(xyz, C.c_float), _p(q, C.c_float), n, p, float(theta), ncrit, mode,
                            _p(cost_a, C.c_double), sp, nout if sample is not None else 0,
                            _p(phi, C.c_double), _p(grad, C.c_double), _p(phases, C.c_double),
                            {"spherical": 0, "cartesian": 1}[basis])
    if not h:
        raise ValueError("non-finite input")
    try:
        tree, tasks = {}, {}
        perm = np.zeros(n, np.int64)
        skeys = np.zeros(n, np.uint64)
        origin = np.zeros(3)
        Lc = np.zeros(1)
        if want_structure:
            nc = L.orc_fmm_ncells(h)
            tree = dict(level=np.zeros(nc, np.int32), prefix=np.zeros(nc, np.uint64),
                        begin=np.zeros(nc, np.int64), count=np.zeros(nc, np.int64))
            if nc:
                L.orc_fmm_tree(h, _p(tree["level"], C.c_int32), _p(tree["prefix"], C.c_uint64),
                               _p(tree["begin"], C.c_int64), _p(tree["count"], C.c_int64))
            nt = L.orc_fmm_ntasks(h)
            tasks = dict(kind=np.zeros(nt, np.int32), tlevel=np.zeros(nt, np.int32),
                         tprefix=np.zeros(nt, np.uint64), slevel=np.zeros(nt, np.int32),
                         sprefix=np.zeros(nt, np.uint64))
            if nt:
                L.orc_fmm_tasks(h, _p(tasks["kind"], C.c_int32), _p(tasks["tlevel"], C.c_int32),
                                _p(tasks["tprefix"], C.c_uint64), _p(tasks["slevel"], C.c_int32),
                                _p(tasks["sprefix"], C.c_uint64))
            L.orc_fmm_perm(h, _p(perm, C.c_int64), _p(skeys, C.c_uint64))
            if n:
                L.orc_fmm_root(h, _p(origin, C.c_double), _p(Lc, C.c_double))
    finally:
        L.orc_fmm_free(h)
    return OracleResult(phi, grad, phases, tree, tasks, perm, skeys, origin, float(Lc[0]))


def direct(xyz, q, targets=None):
    """FP64 O(N^2) direct sum; targets = original indices or None (all)."""
    xyz = np.ascontiguousarray(xyz, np.float32).reshape(-1, 3)
    q = np.ascontiguousarray(q, np.float32)
    if targets is None:
        nt, tp = len(q), None
    else:
        targets = np.ascontiguousarray(targets, np.int64)
        nt, tp = len(targets), _p(targets, C.c_int64)
    phi = np.zeros(nt)
    grad = np.zeros((nt, 3))
    lib().orc_direct(_p(xyz, C.c_float), _p(q, C.c_float), len(q), tp, nt, _p(phi, C.c_double),
                     _p(grad, C.c_double))
    return phi, grad


def canonical_tasks(tasks: dict) -> np.ndarray:
    """Sorted structured array of (kind, tlevel, tprefix, slevel, sprefix)."""
    dt = np.dtype([("kind", np.int32), ("tlevel", np.int32), ("tprefix", np.uint64),
                   ("slevel", np.int32), ("sprefix", np.uint64)])
    a = np.zeros(len(tasks["kind"]), dt)
    for k in dt.names:
        a[k] = tasks[k]
    return np.sort(a, order=list(dt.names))


def rel_l2(a, b):
    """Relative L2 error ||a-b|| / ||b||."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a - b))


def select_kind(mode, cost, nt, ns):
    """The kind the traversal assigns to an accepted pair (DESIGN reading R8)."""
    L = lib()
    L.orc_select_kind.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_int64, C.c_int64]
    L.orc_select_kind.restype = C.c_int
    c = np.ascontiguousarray(cost, np.float64)
    return int(L.orc_select_kind(mode, _p(c, C.c_double), nt, ns))


def task_ranges(res: OracleResult):
    """Map each task to particle ranges: (kind, t_begin, t_count, s_begin, s_count) arrays."""
    tree = res.tree
    key = {(int(l), int(p)): (int(b), int(c)) for l, p, b, c in
           zip(tree["level"], tree["prefix"], tree["begin"], tree["count"])}
    t = res.tasks
    out = np.zeros((len(t["kind"]), 5), np.int64)
    for k in range(len(t["kind"])):
        tb, tc = key[(int(t["tlevel"][k]), int(t["tprefix"][k]))]
        sb, sc = key[(int(t["slevel"][k]), int(t["sprefix"][k]))]
        out[k] = (t["kind"][k], tb, tc, sb, sc)
    return out
