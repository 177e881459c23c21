"""Host logic of the multi-GPU path on CPU (gloo, world_size 2) and the distributed entry points of
the C ABI that need no GPU. The distributed algorithm itself runs in libfmm.so and is tested on the
GPU with an in-process group of ranks (tests/test_gpu_dist.py)."""
import ctypes
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _uid_worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1108_5815_b200.dist import share_unique_id

    # rank 0 stands in for fmm_comm_unique_id with a recognisable pattern
    uid = (np.arange(128) * 7 % 251).astype(np.uint8) if rank == 0 else None
    got = share_unique_id(uid)
    np.save(os.path.join(result_dir, f"u{rank}.npy"), got)
    dist.destroy_process_group()


def test_unique_id_reaches_every_rank(tmp_path):
    # fmm_create_dist needs the same 128-byte NCCL id on every rank (include/fmm.h)
    world = 2
    mp.start_processes(_uid_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    u = [np.load(tmp_path / f"u{r}.npy") for r in range(world)]
    want = (np.arange(128) * 7 % 251).astype(np.uint8)
    assert u[0].dtype == np.uint8 and u[0].shape == (128,)
    assert np.array_equal(u[0], want) and np.array_equal(u[1], want)


def test_distributed_entry_points_validate_without_gpu():
    from paper_1108_5815_b200 import build as fb

    L = ctypes.CDLL(fb.build())
    vp = ctypes.c_void_p
    L.fmm_group_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int]
    L.fmm_group_destroy.argtypes = [vp]
    L.fmm_create_in_group.argtypes = [ctypes.POINTER(vp), ctypes.c_int, ctypes.c_double,
                                      ctypes.c_int, vp, ctypes.c_int]
    L.fmm_create_dist.argtypes = [ctypes.POINTER(vp), ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, vp]
    g = vp()
    assert L.fmm_group_create(ctypes.byref(g), 0) == -1  # at least one rank
    assert L.fmm_group_create(ctypes.byref(g), 17) == -1  # at most 16
    assert L.fmm_group_create(ctypes.byref(g), 3) == 0 and g.value
    h = vp()
    assert L.fmm_create_in_group(ctypes.byref(h), 4, 0.5, 8, None, 0) == -1  # no group
    assert L.fmm_create_in_group(ctypes.byref(h), 0, 0.5, 8, g, 0) == -1  # bad p, no CUDA call
    assert L.fmm_group_destroy(g) == 0
    uid = np.zeros(128, np.uint8)
    assert L.fmm_create_dist(ctypes.byref(h), 4, 0.5, 8, 2, 2, uid.ctypes.data) == -1  # rank >= R
    assert L.fmm_create_dist(ctypes.byref(h), 4, 0.5, 8, 0, 0, uid.ctypes.data) == -1
    assert L.fmm_create_dist(ctypes.byref(h), 4, 0.5, 8, 2, 0, None) == -1
