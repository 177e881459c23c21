"""Multi-GPU evaluation: one process per GPU (PAPER.md:89 spatial domain decomposition).

The distributed algorithm runs inside libfmm.so (fmm_create_dist, include/fmm.h):
the global octree is built from allreduced split bounds, ranks own contiguous Morton runs of whole
leaves, particles move once (alltoallv), multipoles of cells that straddle ranks are allreduced,
and every rank receives exactly the remote multipoles and particles its own interaction lists
name (receiver-driven local essential tree). The collectives are NCCL calls the library issues on
its stream. This module only creates the communicator: rank 0 makes the 128-byte NCCL unique id
and torch.distributed broadcasts it.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .fmm import FMM, nccl_unique_id


def share_unique_id(uid: np.ndarray | None, group=None, device=None) -> np.ndarray:
    """Broadcast rank 0's 128-byte id to every rank of `group` (uint8 tensor; on `device` for an
    NCCL process group, on the CPU for gloo)."""
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) \
            if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if dist.get_rank(group) == 0:
        t.copy_(torch.from_numpy(np.asarray(uid, np.uint8).reshape(128)))
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return t.cpu().numpy()


class DistFMM(FMM):
    """A distributed handle for a torch.distributed job (one rank per GPU). `evaluate(x_local,
    q_local)` is collective and returns (phi, grad) of the rank's own particles, in its order."""

    def __init__(self, p: int = 10, theta: float = 0.4, ncrit: int = 64, mode: str = "hybrid",
                 tune: bool = True, group=None):
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        uid = nccl_unique_id() if rank == 0 else None
        uid = share_unique_id(uid, group)
        super().__init__(p, theta, ncrit, mode, tune, nccl=(world, rank, uid))
        self.world, self.rank = world, rank
