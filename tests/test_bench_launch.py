"""bench.py's multi-GPU launch path on the CPU box: `--gpus N` without torchrun
re-launches itself as N ranks that all join one process group (gloo here, NCCL on the GPU box),
and the N > 1 workloads are the BASELINE ones (C4 strong: the one instance split over the ranks;
C5 weak: 8M per rank)."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus2_launches_two_ranks():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    assert lines[0]["n_gpus"] == 2 and lines[0]["ranks_joined"] == 2
    assert lines[0]["rank_sum"] == 3.0  # ranks 0 and 1 both contributed


def test_strong_and_weak_workloads():
    sys.path.insert(0, ROOT)
    import bench

    world = 4
    shards = [bench.workload("C2", world, r) for r in range(world)]
    n_all = shards[0][2]
    assert n_all == 1_000_000 and all(s[4] == "strong" for s in shards)
    xyz = np.concatenate([s[0] for s in shards])
    from fmm_inputs import make_particles
    ref, _ = make_particles(1_000_000, "uniform", 2)
    assert np.array_equal(xyz, ref)  # the shards are exactly the one C2 instance
    x1, q1, n1, cfg, kind, _ = bench.workload("C4", 1, 0)
    assert n1 == 16_000_000 and len(q1) == n1 and kind == "strong"
