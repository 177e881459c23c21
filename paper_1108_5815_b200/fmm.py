"""ctypes binding of libfmm.so (include/fmm.h). Argument marshalling only: every step of the
method runs in the CUDA kernels behind the C ABI. Torch is used for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
HYBRID, FMM_MODE, TREECODE, DIRECT = 0, 1, 2, 3
MODES = {"hybrid": HYBRID, "fmm": FMM_MODE, "treecode": TREECODE, "direct": DIRECT}
BASES = {"spherical": 0, "cartesian": 1, "auto": 2}
SCHEMES = {"auto": 0, "tc": 1, "gemm": 2, "rotation": 3, "pairs": 4}
SYMBOLS = ["fmm_create", "fmm_destroy", "fmm_evaluate", "fmm_evaluate_ts", "fmm_evaluate_host",
           "fmm_set_stream",
           "fmm_set_mode", "fmm_set_timing", "fmm_set_deterministic", "fmm_set_basis", "fmm_get_basis",
           "fmm_set_m2l_scheme", "fmm_get_m2l_scheme",
           "fmm_tune", "fmm_get_cost_model",
           "fmm_set_cost_model", "fmm_get_stats", "fmm_export_tree", "fmm_export_lists",
           "fmm_export_perm", "fmm_set_partition", "fmm_get_partition", "fmm_partition_indices",
           "fmm_comm_unique_id", "fmm_create_dist", "fmm_group_create", "fmm_group_destroy",
           "fmm_create_in_group", "fmm_strerror", "fmm_last_error"]


class FmmError(RuntimeError):
    pass


class CostModel(C.Structure):
    _fields_ = [("t_pp", C.c_double), ("t_mp", C.c_double), ("t_ml", C.c_double),
                ("p", C.c_int), ("measured", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("n", C.c_int64), ("ncells", C.c_int64), ("nleaves", C.c_int64),
                ("depth", C.c_int32), ("p", C.c_int32),
                ("n_m2l", C.c_int64), ("n_m2p", C.c_int64), ("n_p2p", C.c_int64),
                ("p2p_pairs", C.c_int64), ("m2p_evals", C.c_int64), ("traversal_pairs", C.c_int64),
                ("ms_total", C.c_double), ("ms_tree", C.c_double), ("ms_upward", C.c_double),
                ("ms_traverse", C.c_double), ("ms_m2l", C.c_double), ("ms_p2p", C.c_double),
                ("ms_m2p", C.c_double), ("ms_downward", C.c_double),
                ("launches", C.c_int64), ("cub_calls", C.c_int64),
                ("n_global", C.c_int64), ("rank_lo", C.c_int64), ("rank_hi", C.c_int64),
                ("n_straddle", C.c_int64), ("let_cells", C.c_int64), ("let_particles", C.c_int64),
                ("bytes_sent", C.c_int64), ("ms_comm", C.c_double),
                ("ms_let", C.c_double), ("ms_let_exposed", C.c_double),
                ("ms_p2p_kernel", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def lib_path() -> str:
    return os.environ.get("FMM_LIB", os.path.join(HERE, "libfmm.so"))


_lib = None


def load_library():
    """Load libfmm.so; raises (no fallback) when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        raise FmmError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    vp, i64, dp = C.c_void_p, C.c_int64, C.c_double
    P = C.POINTER
    L.fmm_create.argtypes = [P(vp), C.c_int, dp, C.c_int]
    L.fmm_destroy.argtypes = [vp]
    L.fmm_evaluate.argtypes = [vp, vp, vp, i64, vp, vp]
    L.fmm_evaluate_host.argtypes = [vp, vp, vp, i64, vp, vp]
    L.fmm_evaluate_ts.argtypes = [vp, vp, i64, vp, vp, i64, vp, vp]
    L.fmm_set_stream.argtypes = [vp, vp]
    L.fmm_set_mode.argtypes = [vp, C.c_int]
    L.fmm_set_timing.argtypes = [vp, C.c_int]
    L.fmm_set_deterministic.argtypes = [vp, C.c_int]
    L.fmm_set_m2l_scheme.argtypes = [vp, C.c_int]
    L.fmm_get_m2l_scheme.argtypes = [vp, P(C.c_int), P(dp)]
    L.fmm_set_basis.argtypes = [vp, C.c_int]
    L.fmm_get_basis.argtypes = [vp, P(C.c_int), P(dp), P(dp)]
    L.fmm_tune.argtypes = [vp]
    L.fmm_get_cost_model.argtypes = [vp, P(CostModel)]
    L.fmm_set_cost_model.argtypes = [vp, P(CostModel)]
    L.fmm_get_stats.argtypes = [vp, P(Stats)]
    L.fmm_export_tree.argtypes = [vp, i64, vp, vp, vp, vp, P(i64)]
    L.fmm_export_lists.argtypes = [vp, i64, vp, vp, vp, vp, vp, P(i64)]
    L.fmm_export_perm.argtypes = [vp, i64, vp, vp, vp, vp]
    L.fmm_set_partition.argtypes = [vp, C.c_int, C.c_int]
    L.fmm_get_partition.argtypes = [vp, P(i64), P(i64)]
    L.fmm_partition_indices.argtypes = [vp, vp, i64, P(i64)]
    L.fmm_comm_unique_id.argtypes = [vp]
    L.fmm_create_dist.argtypes = [P(vp), C.c_int, dp, C.c_int, C.c_int, C.c_int, vp]
    L.fmm_group_create.argtypes = [P(vp), C.c_int]
    L.fmm_group_destroy.argtypes = [vp]
    L.fmm_create_in_group.argtypes = [P(vp), C.c_int, dp, C.c_int, vp, C.c_int]
    L.fmm_strerror.argtypes = [C.c_int]
    L.fmm_strerror.restype = C.c_char_p
    L.fmm_last_error.argtypes = [vp]
    L.fmm_last_error.restype = C.c_char_p
    for s in SYMBOLS:
        if s not in ("fmm_strerror", "fmm_last_error"):
            getattr(L, s).restype = C.c_int
    _lib = L
    return L


def _ptr(a) -> int:
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


class LocalGroup:
    """In-process group of `nranks` distributed handles (fmm_group_create): one host thread per
    handle, the ranks may share one GPU. Runs the multi-GPU algorithm on a single device."""

    def __init__(self, nranks: int):
        self.L = load_library()
        g = C.c_void_p()
        rc = self.L.fmm_group_create(C.byref(g), int(nranks))
        if rc != 0:
            raise FmmError(f"fmm_group_create: {self.L.fmm_strerror(rc).decode()}")
        self.g, self.nranks = g, nranks

    def close(self):
        if getattr(self, "g", None):
            self.L.fmm_group_destroy(self.g)
            self.g = None

    __del__ = close


def nccl_unique_id() -> np.ndarray:
    """128-byte NCCL unique id (rank 0 creates it; broadcast it to the other ranks)."""
    L = load_library()
    uid = np.zeros(128, np.uint8)
    rc = L.fmm_comm_unique_id(uid.ctypes.data)
    if rc != 0:
        raise FmmError(f"fmm_comm_unique_id: {L.fmm_strerror(rc).decode()}")
    return uid


class FMM:
    """Handle on the current CUDA device: FMM(p, theta, ncrit, mode='hybrid').

    Distributed handles (fmm.h, multi-GPU): `nccl=(nranks, rank, uid)` joins an NCCL communicator
    (uid from `nccl_unique_id()` on rank 0); `group=(LocalGroup, rank)` joins an in-process group.
    Their `evaluate` is collective and takes / returns the rank's own particle shard."""

    def __init__(self, p: int = 10, theta: float = 0.4, ncrit: int = 64, mode: str = "hybrid",
                 tune: bool = True, nccl=None, group=None):
        self.L = load_library()
        self.p, self.theta, self.ncrit = p, theta, ncrit
        self.distributed = nccl is not None or group is not None
        h = C.c_void_p()
        if not tune:
            os.environ["FMM_NO_TUNE"] = "1"
        try:
            if nccl is not None:
                nr, rk, uid = nccl
                uid = np.ascontiguousarray(np.asarray(uid, np.uint8).reshape(128))
                rc = self.L.fmm_create_dist(C.byref(h), int(p), float(theta), int(ncrit), int(nr),
                                            int(rk), uid.ctypes.data)
                what = "fmm_create_dist"
            elif group is not None:
                grp, rk = group
                rc = self.L.fmm_create_in_group(C.byref(h), int(p), float(theta), int(ncrit),
                                                grp.g, int(rk))
                what = "fmm_create_in_group"
            else:
                rc = self.L.fmm_create(C.byref(h), int(p), float(theta), int(ncrit))
                what = "fmm_create"
        finally:
            if not tune:
                os.environ.pop("FMM_NO_TUNE", None)
        if rc != 0:
            raise FmmError(f"{what}: {self.L.fmm_strerror(rc).decode()}")
        self.h = h
        self.set_mode(mode)

    def _check(self, rc, what):
        if rc != 0:
            msg = self.L.fmm_last_error(self.h).decode()
            raise FmmError(f"{what}: {self.L.fmm_strerror(rc).decode()} ({msg})")

    def close(self):
        if getattr(self, "h", None):
            self.L.fmm_destroy(self.h)
            self.h = None

    __del__ = close

    def set_mode(self, mode):
        m = MODES[mode] if isinstance(mode, str) else int(mode)
        self._check(self.L.fmm_set_mode(self.h, m), "fmm_set_mode")

    def set_timing(self, on: bool):
        self._check(self.L.fmm_set_timing(self.h, int(bool(on))), "fmm_set_timing")

    def set_deterministic(self, on: bool):
        """Bit-reproducible M2L summation order (slower); see fmm_set_deterministic in fmm.h."""
        self._check(self.L.fmm_set_deterministic(self.h, int(bool(on))), "fmm_set_deterministic")

    def set_m2l_scheme(self, scheme):
        """"auto" | "tc" | "gemm" | "rotation" | "pairs" (fmm_set_m2l_scheme)."""
        s = SCHEMES[scheme] if isinstance(scheme, str) else int(scheme)
        self._check(self.L.fmm_set_m2l_scheme(self.h, s), "fmm_set_m2l_scheme")

    def m2l_scheme(self):
        """(scheme in use, {scheme: M2L ms measured by the last tuning})."""
        sc = C.c_int()
        ms = (C.c_double * 5)()
        self._check(self.L.fmm_get_m2l_scheme(self.h, C.byref(sc), ms), "fmm_get_m2l_scheme")
        names = {v: k for k, v in SCHEMES.items()}
        return names[sc.value], {names[i]: ms[i] for i in range(1, 5)}

    def set_basis(self, basis):
        """"spherical" | "cartesian" | "auto" (fmm_set_basis; Cartesian Taylor for p <= 4)."""
        b = BASES[basis] if isinstance(basis, str) else int(basis)
        self._check(self.L.fmm_set_basis(self.h, b), "fmm_set_basis")

    def basis(self):
        """(basis name, auto-switch timings {basis: ms}) of the handle."""
        b, ts, tc = C.c_int(), C.c_double(), C.c_double()
        self._check(self.L.fmm_get_basis(self.h, C.byref(b), C.byref(ts), C.byref(tc)), "fmm_get_basis")
        return {v: k for k, v in BASES.items() if k != "auto"}[b.value], {"spherical": ts.value,
                                                                          "cartesian": tc.value}

    def set_stream(self, stream):
        self._check(self.L.fmm_set_stream(self.h, C.c_void_p(stream)), "fmm_set_stream")

    def tune(self):
        self._check(self.L.fmm_tune(self.h), "fmm_tune")

    def cost_model(self):
        c = CostModel()
        self._check(self.L.fmm_get_cost_model(self.h, C.byref(c)), "fmm_get_cost_model")
        return (c.t_pp, c.t_mp, c.t_ml)

    def set_cost_model(self, t_pp, t_mp, t_ml):
        c = CostModel(float(t_pp), float(t_mp), float(t_ml), int(self.p), 0)
        self._check(self.L.fmm_set_cost_model(self.h, C.byref(c)), "fmm_set_cost_model")

    def stats(self) -> dict:
        s = Stats()
        self._check(self.L.fmm_get_stats(self.h, C.byref(s)), "fmm_get_stats")
        return s.as_dict()

    def evaluate(self, xyz, q, phi=None, grad=None):
        """xyz: CUDA float32 [N,3] contiguous, q: CUDA float32 [N]. Returns (phi [N], grad [N,3])."""
        import torch

        assert xyz.is_cuda and xyz.dtype == torch.float32 and xyz.is_contiguous()
        assert q.is_cuda and q.dtype == torch.float32 and q.is_contiguous()
        n = q.numel()
        if phi is None:
            phi = torch.empty(n, dtype=torch.float32, device=xyz.device)
        if grad is None:
            grad = torch.empty((n, 3), dtype=torch.float32, device=xyz.device)
        if n == 0 and not self.distributed:
            return phi, grad
        self._check(self.L.fmm_set_stream(self.h, C.c_void_p(torch.cuda.current_stream().cuda_stream)),
                    "fmm_set_stream")
        self._check(self.L.fmm_evaluate(self.h, xyz.data_ptr(), q.data_ptr(), n, phi.data_ptr(),
                                        grad.data_ptr()), "fmm_evaluate")
        return phi, grad

    def evaluate_ts(self, xyz_t, xyz_s, q_s):
        """Distinct targets and sources (fmm_evaluate_ts): CUDA float32 xyz_t [Nt,3], xyz_s [Ns,3],
        q_s [Ns]. Returns (phi [Nt], grad [Nt,3]) at the targets due to the sources."""
        import torch

        for a in (xyz_t, xyz_s, q_s):
            assert a.is_cuda and a.dtype == torch.float32 and a.is_contiguous()
        nt, ns = xyz_t.shape[0], q_s.numel()
        phi = torch.empty(nt, dtype=torch.float32, device=xyz_t.device)
        grad = torch.empty((nt, 3), dtype=torch.float32, device=xyz_t.device)
        if nt == 0:
            return phi, grad
        self._check(self.L.fmm_set_stream(self.h, C.c_void_p(torch.cuda.current_stream().cuda_stream)),
                    "fmm_set_stream")
        self._check(self.L.fmm_evaluate_ts(self.h, xyz_t.data_ptr(), nt, xyz_s.data_ptr() if ns else None,
                                           q_s.data_ptr() if ns else None, ns, phi.data_ptr(),
                                           grad.data_ptr()), "fmm_evaluate_ts")
        return phi, grad

    def evaluate_host(self, xyz: np.ndarray, q: np.ndarray, phi=None, grad=None):
        """Host (numpy, ideally pinned) buffers: H2D + evaluate + D2H inside the C ABI call."""
        xyz = np.ascontiguousarray(xyz, np.float32)
        q = np.ascontiguousarray(q, np.float32)
        n = len(q)
        phi = np.empty(n, np.float32) if phi is None else phi
        grad = np.empty((n, 3), np.float32) if grad is None else grad
        self._check(self.L.fmm_evaluate_host(self.h, _ptr(xyz), _ptr(q), n, _ptr(phi), _ptr(grad)),
                    "fmm_evaluate_host")
        return phi, grad

    def set_partition(self, nparts: int, part: int):
        self._check(self.L.fmm_set_partition(self.h, int(nparts), int(part)), "fmm_set_partition")

    def partition_range(self):
        lo, hi = C.c_int64(), C.c_int64()
        self._check(self.L.fmm_get_partition(self.h, C.byref(lo), C.byref(hi)), "fmm_get_partition")
        return lo.value, hi.value

    def partition_indices(self, device=None):
        """Caller indices (int64 CUDA tensor) of the particles evaluated by this partition."""
        import torch

        lo, hi = self.partition_range()
        out = torch.empty(max(hi - lo, 1), dtype=torch.int64, device=device or "cuda")
        cnt = C.c_int64()
        self._check(self.L.fmm_partition_indices(self.h, out.data_ptr(), out.numel(), C.byref(cnt)),
                    "fmm_partition_indices")
        return out[: cnt.value]

    def export_tree(self) -> dict:
        cnt = C.c_int64()
        self.L.fmm_export_tree(self.h, 0, None, None, None, None, C.byref(cnt))
        n = cnt.value
        t = dict(level=np.zeros(n, np.int32), prefix=np.zeros(n, np.uint64),
                 begin=np.zeros(n, np.int64), count=np.zeros(n, np.int64))
        self._check(self.L.fmm_export_tree(self.h, n, _ptr(t["level"]), _ptr(t["prefix"]),
                                           _ptr(t["begin"]), _ptr(t["count"]), C.byref(cnt)),
                    "fmm_export_tree")
        return t

    def export_lists(self) -> dict:
        cnt = C.c_int64()
        self.L.fmm_export_lists(self.h, 0, None, None, None, None, None, C.byref(cnt))
        n = cnt.value
        t = dict(kind=np.zeros(n, np.int32), tlevel=np.zeros(n, np.int32),
                 tprefix=np.zeros(n, np.uint64), slevel=np.zeros(n, np.int32),
                 sprefix=np.zeros(n, np.uint64))
        self._check(self.L.fmm_export_lists(self.h, n, _ptr(t["kind"]), _ptr(t["tlevel"]),
                                            _ptr(t["tprefix"]), _ptr(t["slevel"]),
                                            _ptr(t["sprefix"]), C.byref(cnt)), "fmm_export_lists")
        return t

    def export_perm(self, n: int):
        perm = np.zeros(n, np.int64)
        keys = np.zeros(n, np.uint64)
        origin = np.zeros(3)
        Lside = np.zeros(1)
        self._check(self.L.fmm_export_perm(self.h, n, _ptr(perm), _ptr(keys), _ptr(origin),
                                           _ptr(Lside)), "fmm_export_perm")
        return perm, keys, origin, float(Lside[0])
