"""Multi-GPU evaluation: one process per GPU, torch.distributed (NCCL) for the plumbing.

PAPER.md:89 distributes the FMM by spatial domain decomposition. SURVEY §8(e) plans a Morton
partition with a local-essential-tree (LET) exchange. Round 1 ships the first step of that plan:

1. Every rank contributes its local particle shard. An all-gather over NVLink builds the global
   particle set on every rank; this is the one exchange of the data path.
2. Every rank builds the global tree and runs the upward sweep over all particles. This part is
   redundant across ranks; the LET exchange replaces it next.
3. Every rank evaluates only the targets of its Morton part (`fmm_set_partition`). Those are the
   leaves whose first sorted particle index b has floor(b * world / N) == rank. Traversal, M2L,
   P2P, M2P and the downward sweep are therefore split across ranks.
4. The results go back to the ranks that own the particles with one all-to-all.

All arithmetic runs in libfmm.so. This module only moves tensors: all_gather, index_select and
all_to_all_single on the device.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def gather_particles(x_local: torch.Tensor, q_local: torch.Tensor, group=None):
    """All-gather uneven shards. Returns (xyz [N,3], q [N], offsets [world+1] int64 on the device)."""
    world = dist.get_world_size(group)
    dev = x_local.device
    n_loc = torch.tensor([q_local.numel()], dtype=torch.int64, device=dev)
    counts = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(counts, n_loc, group=group)
    nmax = int(counts.max().item())
    xp = torch.zeros((nmax, 4), dtype=torch.float32, device=dev)
    xp[: q_local.numel(), :3] = x_local
    xp[: q_local.numel(), 3] = q_local
    allp = torch.empty((world * nmax, 4), dtype=torch.float32, device=dev)
    dist.all_gather_into_tensor(allp, xp, group=group)
    offsets = torch.zeros(world + 1, dtype=torch.int64, device=dev)
    offsets[1:] = torch.cumsum(counts, 0)
    if int(counts.min().item()) == nmax:
        g = allp
    else:
        keep = torch.cat([torch.arange(r * nmax, r * nmax + int(c), device=dev)
                          for r, c in enumerate(counts.tolist())])
        g = allp.index_select(0, keep)
    return g[:, :3].contiguous(), g[:, 3].contiguous(), offsets


def route_results(idx: torch.Tensor, vals: torch.Tensor, offsets: torch.Tensor, n_local: int,
                  group=None):
    """Send the rows of vals, computed here for global particle indices idx, to the ranks that own
    those particles; return this rank's rows [n_local, k] in its local particle order."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dest = torch.bucketize(idx, offsets[1:], right=True)
    order = torch.argsort(dest, stable=True)
    idx, vals, dest = idx[order], vals[order], dest[order]
    send = torch.bincount(dest, minlength=world).to(torch.int64)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    s_list, r_list = send.tolist(), recv.tolist()
    ridx = torch.empty(sum(r_list), dtype=idx.dtype, device=idx.device)
    rval = torch.empty((sum(r_list), vals.shape[1]), dtype=vals.dtype, device=vals.device)
    dist.all_to_all_single(ridx, idx, r_list, s_list, group=group)
    dist.all_to_all_single(rval, vals.contiguous(), r_list, s_list, group=group)
    out = torch.zeros((n_local, vals.shape[1]), dtype=vals.dtype, device=vals.device)
    out[ridx - offsets[rank]] = rval
    return out


def broadcast_cost_model(fmm, group=None, src: int = 0):
    """Give every rank rank `src`'s measured cost table (the kind choice of a
    pair must not depend on which rank evaluates it, so that the union of the per-rank lists is
    the one-GPU list set)."""
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")
    t = torch.tensor(list(fmm.cost_model()), dtype=torch.float64, device=dev)
    dist.broadcast(t, src=src, group=group)
    fmm.set_cost_model(*[float(v) for v in t.tolist()])


class DistFMM:
    """Wraps a single-GPU `FMM` handle for a torch.distributed job (one rank per GPU)."""

    def __init__(self, fmm, world: int, rank: int, group=None, share_cost_model: bool = True):
        self.f, self.world, self.rank, self.group = fmm, world, rank, group
        self.f.set_partition(world, rank)
        if share_cost_model and world > 1:
            broadcast_cost_model(self.f, group)

    def __getattr__(self, name):  # set_timing, stats, cost_model, ... of the local handle
        return getattr(self.f, name)

    def evaluate(self, x_local: torch.Tensor, q_local: torch.Tensor):
        xg, qg, offsets = gather_particles(x_local, q_local, self.group)
        n = qg.numel()
        phi = torch.empty(n, dtype=torch.float32, device=xg.device)
        grad = torch.empty((n, 3), dtype=torch.float32, device=xg.device)
        self.f.evaluate(xg, qg, phi, grad)
        idx = self.f.partition_indices(device=xg.device)
        vals = torch.cat([phi.index_select(0, idx)[:, None], grad.index_select(0, idx)], 1)
        out = route_results(idx, vals, offsets, q_local.numel(), self.group)
        return out[:, 0].contiguous(), out[:, 1:].contiguous()
