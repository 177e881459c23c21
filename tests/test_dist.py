"""Multi-process host logic of the multi-GPU path (paper_1108_5815_b200/dist.py) with gloo on CPU,
world_size 2: particle all-gather, the Morton target partition rule of fmm_set_partition (include/
fmm.h) and result routing; the per-rank evaluation is the FP64 oracle's direct sum on the part's
targets, so every particle must come back exactly once with its direct-sum value."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from fmm_inputs import make_particles
    from oracle import oracle as O
    from paper_1108_5815_b200.dist import gather_particles, route_results

    n_local = 700 + 311 * rank  # uneven shards
    xyz, q = make_particles(n_local, "plummer", 40 + rank)
    X, Q = torch.from_numpy(xyz), torch.from_numpy(q)
    xg, qg, offsets = gather_particles(X, Q)
    N = qg.numel()
    # the Morton target partition of fmm_set_partition, on the oracle's tree
    ref = O.fmm(xg.numpy(), qg.numpy(), 2, 0.5, 16, O.FMM)
    leaves = [(int(b), int(c)) for l, p, b, c in zip(ref.tree["level"], ref.tree["prefix"],
                                                      ref.tree["begin"], ref.tree["count"])
              if not any((l + 1, p * 8 + o) in {(int(a), int(b2)) for a, b2 in
                                                 zip(ref.tree["level"], ref.tree["prefix"])}
                         for o in range(8))]
    mine = [(b, c) for b, c in leaves if (b * world) // N == rank]
    sorted_idx = np.concatenate([np.arange(b, b + c) for b, c in mine]) if mine else np.zeros(0, int)
    idx = torch.from_numpy(ref.perm[sorted_idx].astype(np.int64))
    phi, grad = O.direct(xg.numpy(), qg.numpy(), idx.numpy())
    vals = torch.from_numpy(np.concatenate([phi[:, None], grad], 1))
    out = route_results(idx, vals, offsets, n_local)
    full = O.direct(xg.numpy(), qg.numpy())
    lo = int(offsets[rank])
    np.save(os.path.join(result_dir, f"r{rank}.npy"),
            np.stack([np.abs(out[:, 0].numpy() - full[0][lo:lo + n_local]).max(),
                      np.abs(out[:, 1:].numpy() - full[1][lo:lo + n_local]).max(),
                      float(len(idx)), float(N)]))
    dist.destroy_process_group()


def test_gather_partition_route_world2(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    res = [np.load(tmp_path / f"r{r}.npy") for r in range(world)]
    N = res[0][3]
    assert sum(r[2] for r in res) == N  # every target evaluated by exactly one rank
    for r in res:
        assert r[0] == 0.0 and r[1] == 0.0  # routed rows are the owner's rows, bit for bit


class _FakeHandle:
    """Stands in for FMM: only the cost-table accessors broadcast_cost_model uses."""

    def __init__(self, c):
        self.c = tuple(c)

    def cost_model(self):
        return self.c

    def set_cost_model(self, *c):
        self.c = tuple(c)


def _cost_worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1108_5815_b200.dist import broadcast_cost_model

    h = _FakeHandle((1.0e-12 * (rank + 1), 3.0e-10 * (rank + 1), 7.0e-9 * (rank + 1)))
    broadcast_cost_model(h)
    np.save(os.path.join(result_dir, f"c{rank}.npy"), np.array(h.c))
    dist.destroy_process_group()


def test_cost_table_is_rank0s_on_every_rank(tmp_path):
    # one cost table for all ranks, or the kind choice of a pair would depend
    # on the rank that evaluates it
    world = 2
    mp.start_processes(_cost_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    c = [np.load(tmp_path / f"c{r}.npy") for r in range(world)]
    assert np.array_equal(c[0], c[1]) and np.array_equal(c[0], [1.0e-12, 3.0e-10, 7.0e-9])
