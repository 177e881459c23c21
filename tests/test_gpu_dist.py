"""GPU tests of the distributed evaluation (include/fmm.h multi-GPU section): R ranks
as an in-process group on one GPU (fmm_group_create / fmm_create_in_group, one host thread per
rank). The algorithm and every kernel are those of the NCCL path; only the transport differs.

Bars: the global tree of every rank equals the single-GPU tree bit for bit; the union of the
per-rank interaction lists equals the single-GPU lists (as a set, no rank listing a pair twice);
phi / grad of every particle match the single-GPU evaluation and the FP64 oracle within 1e-5
relative L2 (SURVEY §8(c) bar), whatever the initial (random, uneven) distribution of particles.
"""
import threading

import numpy as np
import pytest

from fmm_inputs import make_particles

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_1108_5815_b200 import FMM  # noqa: E402
from paper_1108_5815_b200.fmm import LocalGroup  # noqa: E402

COST = (2e-12, 6e-11, 2.5e-9)


@pytest.fixture(autouse=True)
def let_check(monkeypatch):
    """Every distributed evaluation verifies that its local essential tree is complete (each
    remote multipole and particle range its lists name was received; FMM_LET_CHECK)."""
    monkeypatch.setenv("FMM_LET_CHECK", "1")


def shards(n, R, seed, empty_rank=None):
    """Random, uneven assignment of the particle indices to R ranks (optionally one empty)."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    w = rng.uniform(0.3, 1.7, R)
    if empty_rank is not None:
        w[empty_rank] = 0.0
    cuts = np.floor(np.cumsum(w) / w.sum() * n).astype(int)
    cuts[-1] = n
    return np.split(perm, cuts[:-1])


def run_group(R, xyz, q, parts, p, theta, ncrit, mode, evals=1, timing=False):
    grp = LocalGroup(R)
    out = [None] * R
    errs = []

    def worker(r):
        f = None
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                f = FMM(p=p, theta=theta, ncrit=ncrit, mode=mode, tune=False, group=(grp, r))
                f.set_cost_model(*COST)
                f.set_timing(timing)
                x = torch.from_numpy(np.ascontiguousarray(xyz[parts[r]])).cuda()
                c = torch.from_numpy(np.ascontiguousarray(q[parts[r]])).cuda()
                for _ in range(evals):
                    phi, grad = f.evaluate(x, c)
                s.synchronize()
                out[r] = dict(phi=phi.cpu().numpy().astype(np.float64),
                              grad=grad.cpu().numpy().astype(np.float64),
                              lists=f.export_lists(), tree=f.export_tree(), stats=f.stats())
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))
        finally:
            if f is not None:
                f.close()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a rank hung"
    grp.close()
    assert not errs, errs
    return out


def single(xyz, q, p, theta, ncrit, mode):
    f = FMM(p=p, theta=theta, ncrit=ncrit, mode=mode, tune=False)
    f.set_cost_model(*COST)
    phi, grad = f.evaluate(torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda())
    torch.cuda.synchronize()
    res = dict(phi=phi.cpu().numpy().astype(np.float64), grad=grad.cpu().numpy().astype(np.float64),
               lists=f.export_lists(), tree=f.export_tree())
    f.close()
    return res


def as_set(lists):
    c = O.canonical_tasks(lists)
    return c, {tuple(r) for r in c.tolist()}


CASES = [  # (R, dist, n, p, theta, ncrit, mode, empty rank)
    (2, "uniform", 20000, 6, 0.5, 32, "hybrid", None),
    (3, "plummer", 30000, 8, 0.45, 32, "hybrid", None),
    (4, "uniform", 12000, 5, 0.4, 16, "fmm", 2),
    (4, "plummer", 16000, 6, 0.5, 24, "treecode", None),
    (2, "mixed", 5000, 10, 0.4, 64, "hybrid", 0),
]


@pytest.mark.parametrize("let", ["send", "recv"])
@pytest.mark.parametrize("R,dist,n,p,theta,ncrit,mode,empty", CASES)
def test_dist_equals_single_gpu(monkeypatch, R, dist, n, p, theta, ncrit, mode, empty, let):
    """Both local-essential-tree exchanges: the sender-side one (default; overlaps the traversal)
    and the round-1 receiver-driven one (FMM_LET=recv)."""
    monkeypatch.setenv("FMM_LET", let)
    xyz, q = make_particles(n, dist, 50 + R)
    parts = shards(n, R, 7 + R, empty)
    ref = single(xyz, q, p, theta, ncrit, mode)
    out = run_group(R, xyz, q, parts, p, theta, ncrit, mode)
    # the global tree on every rank
    for o in out:
        for k in ("level", "prefix", "begin", "count"):
            assert np.array_equal(o["tree"][k], ref["tree"][k]), k
    # lists: union over the ranks = single-GPU lists; no rank lists a pair twice
    _, ref_set = as_set(ref["lists"])
    union = set()
    for o in out:
        c, s = as_set(o["lists"])
        assert len(s) == len(c)
        union |= s
    assert union == ref_set
    # fields, back in every rank's own order
    phi = np.zeros(n)
    grad = np.zeros((n, 3))
    for r, o in enumerate(out):
        assert o["phi"].shape == (len(parts[r]),)
        phi[parts[r]] = o["phi"]
        grad[parts[r]] = o["grad"]
    assert O.rel_l2(phi, ref["phi"]) < 1e-6 and O.rel_l2(grad, ref["grad"]) < 1e-6
    orc = O.fmm(xyz, q, p, theta, ncrit, {"hybrid": O.HYBRID, "fmm": O.FMM, "treecode": O.TREECODE}[mode],
                cost=COST)
    assert O.rel_l2(phi, orc.phi) < 1e-5 and O.rel_l2(grad, orc.grad) < 1e-5
    # every rank's targets are whole leaves and the ranges tile [0, N)
    lo = sorted((o["stats"]["rank_lo"], o["stats"]["rank_hi"]) for o in out)
    assert lo[0][0] == 0 and lo[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(lo, lo[1:]))
    if R > 1:
        assert sum(o["stats"]["let_cells"] + o["stats"]["let_particles"] for o in out) > 0


def test_dist_repeated_and_single_rank():
    # a 1-rank group is the single-GPU path with a trivial exchange; repeated evaluations reuse
    # the grown buffers
    xyz, q = make_particles(6000, "plummer", 77)
    ref = single(xyz, q, 6, 0.5, 32, "hybrid")
    out = run_group(1, xyz, q, [np.arange(6000)], 6, 0.5, 32, "hybrid", evals=2)
    assert O.rel_l2(out[0]["phi"], ref["phi"]) < 1e-6
    out = run_group(3, xyz, q, shards(6000, 3, 1), 6, 0.5, 32, "hybrid", evals=3)
    assert out[0]["stats"]["n_global"] == 6000


def test_dist_bench_workload_shape():
    # bench.py at N > 1 (C4 strong scaling): ONE uniform instance split evenly over the ranks,
    # p = 10, theta = 0.4, ncrit = 64, here 2 x 200k; the sender-side exchange is timed on its
    # own stream and reported with how much of it the traversal did not hide
    R, n = 2, 400_000
    xyz, q = make_particles(n, "uniform", 4)
    parts = [np.arange(r * n // R, (r + 1) * n // R) for r in range(R)]
    ref = single(xyz, q, 10, 0.4, 64, "hybrid")
    out = run_group(R, xyz, q, parts, 10, 0.4, 64, "hybrid", evals=2, timing=True)
    phi = np.concatenate([o["phi"] for o in out])
    grad = np.concatenate([o["grad"] for o in out])
    assert O.rel_l2(phi, ref["phi"]) < 1e-6 and O.rel_l2(grad, ref["grad"]) < 1e-6
    s = np.random.default_rng(3).choice(len(q), 512, replace=False)
    d = O.direct(xyz, q, s)
    assert O.rel_l2(phi[s], d[0]) < 1e-4 and O.rel_l2(grad[s], d[1]) < 1e-3
    st = [o["stats"] for o in out]
    assert all(x["let_cells"] > 0 and x["let_particles"] > 0 for x in st)
    assert all(x["ms_let"] > 0 and 0 <= x["ms_let_exposed"] <= x["ms_let"] + 1e-3 for x in st)


def test_nccl_transport_world1(tmp_path):
    # the NCCL transport (fmm_comm_unique_id / fmm_create_dist, libnccl dlopen'ed) end to end
    # through paper_1108_5815_b200.dist.DistFMM on a 1-rank torch.distributed NCCL group: the
    # distributed pipeline with its exchanges against the plain handle
    import socket

    import torch.distributed as dist

    from paper_1108_5815_b200.dist import DistFMM

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        xyz, q = make_particles(30000, "plummer", 91)
        ref = single(xyz, q, 8, 0.45, 32, "hybrid")
        f = DistFMM(p=8, theta=0.45, ncrit=32, mode="hybrid", tune=False)
        f.set_cost_model(*COST)
        phi, grad = f.evaluate(torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda())
        torch.cuda.synchronize()
        st = f.stats()
        f.close()
    finally:
        dist.destroy_process_group()
    assert O.rel_l2(phi.cpu().numpy(), ref["phi"]) < 1e-6
    assert O.rel_l2(grad.cpu().numpy(), ref["grad"]) < 1e-6
    assert st["n_global"] == 30000 and st["rank_lo"] == 0 and st["rank_hi"] == 30000


def test_dist_nonfinite_fails_on_every_rank():
    # a NaN on one rank: the non-finite flag travels with the bbox allreduce, so every rank
    # returns FMM_E_NONFINITE at the same point (no rank is left waiting in a collective), and
    # the group is usable again afterwards
    from paper_1108_5815_b200 import FmmError

    R = 3
    xyz, q = make_particles(9000, "uniform", 3)
    parts = shards(9000, R, 4)
    bad = xyz.copy()
    bad[parts[1][5], 2] = np.nan
    grp = LocalGroup(R)
    errs, ok = [None] * R, [None] * R

    def worker(r):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            f = FMM(p=4, theta=0.5, ncrit=16, tune=False, group=(grp, r))
            f.set_cost_model(*COST)
            try:
                f.evaluate(torch.from_numpy(bad[parts[r]]).cuda(), torch.from_numpy(q[parts[r]]).cuda())
            except FmmError as e:
                errs[r] = str(e)
            phi, _ = f.evaluate(torch.from_numpy(xyz[parts[r]]).cuda(), torch.from_numpy(q[parts[r]]).cuda())
            s.synchronize()
            ok[r] = phi.cpu().numpy()
            f.close()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "a rank hung"
    grp.close()
    assert all(e is not None and "non-finite" in e for e in errs), errs
    ref = single(xyz, q, 4, 0.5, 16, "hybrid")
    phi = np.zeros(9000)
    for r in range(R):
        phi[parts[r]] = ok[r]
    assert O.rel_l2(phi, ref["phi"]) < 1e-6
