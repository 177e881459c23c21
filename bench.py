#!/usr/bin/env python
"""bench.py — FMM time-to-solution on B200 (BASELINE.json metric), driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4|C5]

Workload at N=1: BASELINE.json configs[3] = C4, the configuration the metric ("at 1/2/4/8
B200") is quoted on and the largest single-GPU one: N = 16,000,000 uniform random charges in the
unit cube, Laplace potential + gradient, p = 10, theta = 0.4, ncrit = 64, hybrid M2L/M2P/P2P choice
auto-tuned on the device. One step = one full fmm_evaluate (tree build, upward
sweep, traversal, M2L/M2P/P2P, downward sweep) on inputs already resident in HBM (256 MB of
inputs, larger than the 126 MB L2; L2 is also flushed with a 512 MiB write before every timed
step, outside the timed interval). `value` = particles evaluated per second over all ranks
(N / time-to-solution). C2 (1M uniform) and C3 (4M Plummer) are timed too, as extra fields with
their own clock records, and so is the deterministic (bit-reproducible) M2L summation mode.

N > 1: one process per GPU. Without torchrun in the environment, `--gpus N` re-launches itself
under `python -m torch.distributed.run --nproc-per-node N` (127.0.0.1). Default: C4 STRONG
scaling (the 16M-particle instance split evenly over the ranks, one distributed handle per rank:
fmm_create_dist, NCCL inside libfmm.so); `--config C5`: WEAK scaling, 8M particles
per rank (seed 5 + rank, one global uniform problem of N x 8M). Max over ranks; rank 0 prints.

`--impl reference` times the CPU FP64 oracle (oracle/, the only other arm this tier has) on the
host cores: each step is the full oracle FMM of a bounded sub-box of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from fmm_inputs import CONFIGS, make_particles  # noqa: E402

METRIC = "FMM time-to-solution & P2P/M2L Gflop/s vs FP32 peak at 1/2/4/8 B200"
UNIT = "particles/s"
FP32_LANES_PER_SM = 128
N_SM = 148
# 19 flop + 1 rsqrt per pair (3 sub for d, 5 for r^2, 1 q/r, 1 phi add, 2 for
# q/r^3, 6 for the three gradient FMAs; the rsqrt is counted as 1)
P2P_FLOP_PER_PAIR = 19
# cpu_baseline: a bounded sub-box of the benchmarked C4 instance (same density, same leaf
# occupancy): [0,.5) x [0,.5) x [0,.25), about 1M particles, 10-30 s of the FP64 oracle on 16 cores
CPU_SUBBOX = (0.5, 0.5, 0.25)
# --impl reference steps: [0,.25) x [0,.25) x [0,.125) of C4, about 125k particles per step
REF_SUBBOX = (0.25, 0.25, 0.125)


def m2l_flops(p: int) -> int:
    """Algorithmic M2L work per cell pair: the translation as a real (p+1)^2 x (p+1)^2 matrix
    (real degrees of freedom of a real field) applied to the source multipole, 2 (p+1)^4 flop.
    (The paper's complex double loop over signed orders is 8 NC(p) (p+1)^2 = 63,888 at p=10.)"""
    return 2 * (p + 1) ** 4


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def make_handle(cfg, mode="hybrid", deterministic=False, distributed=False):
    """The handle exactly as the benchmark uses it (tests/test_gpu_parity.py builds it with this
    same function). Accumulate mode (M2L results reduced in L2, unordered): created without the
    default-mode tuning, switched, then tuned, so the kernel pre-calculation times
    the M2L path the evaluations use. Deterministic mode: the library default, tuned at creation."""
    if distributed:
        from paper_1108_5815_b200.dist import DistFMM as cls
    else:
        from paper_1108_5815_b200 import FMM as cls
    f = cls(p=cfg["p"], theta=cfg["theta"], ncrit=cfg["ncrit"], mode=mode, tune=deterministic)
    f.set_deterministic(deterministic)
    if not deterministic:
        f.tune()
    return f


def subbox(xyz, q, box):
    m = np.all(xyz < np.asarray(box, np.float32), axis=1)
    return np.ascontiguousarray(xyz[m]), np.ascontiguousarray(q[m])


def workload(config, world, rank):
    """(xyz, q) of this rank, total particle count, config dict, scaling kind, description."""
    cfg = dict(CONFIGS[config])
    if config == "C5":  # weak: 8M per rank, one global uniform problem of world x 8M
        xyz, q = make_particles(cfg["n"], cfg["dist"], cfg["seed"] + rank)
        q = (q / world).astype(np.float32)  # q = 1/N_global
        desc = (f"C5 weak scaling: {cfg['n'] // 10**6}M uniform particles per GPU "
                f"({world} x {cfg['n'] // 10**6}M = {world * cfg['n'] / 1e6:g}M in one problem), "
                f"p={cfg['p']}, theta={cfg['theta']}, ncrit={cfg['ncrit']}, auto-tuned hybrid")
        return xyz, q, cfg["n"] * world, cfg, "weak", desc
    xyz, q = make_particles(cfg["n"], cfg["dist"], cfg["seed"])
    desc = (f"{config}: N={cfg['n'] / 1e6:g}M {cfg['dist']}, Laplace phi+grad, p={cfg['p']}, "
            f"theta={cfg['theta']}, ncrit={cfg['ncrit']}, auto-tuned hybrid")
    if world > 1:  # strong: the one instance split evenly over the ranks (any shard works)
        lo, hi = rank * cfg["n"] // world, (rank + 1) * cfg["n"] // world
        xyz, q = np.ascontiguousarray(xyz[lo:hi]), np.ascontiguousarray(q[lo:hi])
        desc += f", strong scaling over {world} GPUs"
    # the total is fixed as N grows: strong scaling (at N = 1 too, so the N = 1..8 lines agree)
    return xyz, q, cfg["n"], cfg, "strong", desc


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def cpu_baseline(cost, cfg, mode_name):
    """The FP64 oracle as it stands, on this host's cores (rank 0, N=1 only): the full oracle FMM
    of a bounded sub-box of the benchmarked C4 instance."""
    from oracle import oracle as O

    xyz, q = make_particles(cfg["n"], cfg["dist"], cfg["seed"])
    xyz, q = subbox(xyz, q, CPU_SUBBOX)
    mode = {"hybrid": O.HYBRID, "fmm": O.FMM, "treecode": O.TREECODE}[mode_name]
    t = time.perf_counter()
    O.fmm(xyz, q, cfg["p"], cfg["theta"], cfg["ncrit"], mode, cost=cost, want_structure=False)
    dt = time.perf_counter() - t
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": len(q) / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "seconds": dt, "n": len(q),
            "sample": f"full oracle FMM (FP64, OpenMP) of the {len(q)} particles of the C4 instance "
                      f"in [0,{CPU_SUBBOX[0]})x[0,{CPU_SUBBOX[1]})x[0,{CPU_SUBBOX[2]}) (1/16 of C4, "
                      f"same density and leaf occupancy; p={cfg['p']}, theta={cfg['theta']}, "
                      f"ncrit={cfg['ncrit']}, {mode_name}, the GPU's measured cost model)"}


def run_reference(args):
    """--impl reference: the CPU oracle arm (rank 0 only; other ranks exit without work)."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    from oracle import oracle as O

    cfg = CONFIGS["C4"]
    xyz, q = make_particles(cfg["n"], cfg["dist"], cfg["seed"])
    xyz, q = subbox(xyz, q, REF_SUBBOX)
    n = len(q)
    cost = (5.6e-13, 1.2e-10, 2.2e-10)  # the B200 cost model fmm_tune measures (accumulate mode)
    times = []
    for it in range(args.warmup + args.steps):
        t = time.perf_counter()
        O.fmm(xyz, q, cfg["p"], cfg["theta"], cfg["ncrit"], O.HYBRID, cost=cost, want_structure=False)
        if it >= args.warmup:
            times.append(time.perf_counter() - t)
    ms = 1e3 * sum(times) / len(times)
    value = n / (ms * 1e-3)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C4 recipe, bounded sub-box [0,{REF_SUBBOX[0]})x[0,{REF_SUBBOX[1]})"
                               f"x[0,{REF_SUBBOX[2]}) of the C4 instance: N={n}",
                   "n": n, "p": cfg["p"], "theta": cfg["theta"], "ncrit": cfg["ncrit"], "mode": "hybrid"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"each step: full FP64 oracle FMM of the {n} C4 particles in the sub-box, "
                                   "on the host cores"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch(args):
    """`--gpus N` without torchrun: re-run this script as N ranks (one per GPU) and return the
    launcher's exit code. Rank 0's JSON line is the only stdout line the ranks print."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def run_dry(args):
    """--dry-run: the multi-rank launch path without the FMM (CPU box: gloo). Every rank joins the
    process group and contributes its rank; rank 0 prints what it saw."""
    import torch
    import torch.distributed as dist

    world, rank = env_int("WORLD_SIZE", 1), env_int("RANK", 0)
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    if world > 1:
        dist.init_process_group(backend, rank=rank, world_size=world)
        t = torch.tensor([rank + 1.0, 1.0])
        if backend == "nccl":
            torch.cuda.set_device(env_int("LOCAL_RANK", 0))
            t = t.cuda()
        dist.all_reduce(t)
        ranks, seen = int(t[1].item()), float(t[0].item())
        dist.destroy_process_group()
    else:
        ranks, seen = 1, 1.0
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_joined": ranks,
                          "rank_sum": seen, "backend": backend if world > 1 else None,
                          "config": args.config}), flush=True)


def time_steps(f, X, Q, steps, barrier, flush, stream, local):
    """`steps` evaluations bracketed by barrier + synchronize, each timed with CUDA events on the
    launching stream, L2 flushed before each; per-phase CUDA-event times summed."""
    import torch

    step_ms = []
    phase = {k: 0.0 for k in ("ms_m2l", "ms_p2p", "ms_p2p_kernel", "ms_m2p", "ms_tree",
                              "ms_upward", "ms_traverse", "ms_downward")}
    launches = 0
    f.set_timing(True)
    with ClockSampler(local) as clk:
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/": the launch list
        for _ in range(steps):
            flush.fill_(1.0)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            f.evaluate(X, Q)
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            s = f.stats()
            for k in phase:
                phase[k] += s[k]
            launches += s["launches"]
        torch.cuda.nvtx.range_pop()
        barrier()
    f.set_timing(False)
    return step_ms, {k: v / steps for k, v in phase.items()}, launches / steps, clk.summary()


def extra_config(name, mode, steps, warmup, flush, stream, local):
    """C2 / C3 on one GPU: the same handle recipe, its own steps and clock record."""
    import torch

    cfg = CONFIGS[name]
    xyz, q = make_particles(cfg["n"], cfg["dist"], cfg["seed"])
    X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
    f = make_handle(cfg, mode, False)
    try:
        for _ in range(warmup):
            f.evaluate(X, Q)
        ms, ph, _, clk = time_steps(f, X, Q, steps, torch.cuda.synchronize, flush, stream, local)
        st = f.stats()
    finally:
        f.close()
    t = sum(ms) / len(ms)
    return {"workload": f"{name}: N={cfg['n'] / 1e6:g}M {cfg['dist']}, p={cfg['p']}, "
                        f"theta={cfg['theta']}, ncrit={cfg['ncrit']}, auto-tuned hybrid",
            "ms_per_step": t, "value": cfg["n"] / (t * 1e-3), "unit": UNIT, "steps": steps,
            "phases_ms": ph, "counts": {k: st[k] for k in ("ncells", "nleaves", "depth", "n_m2l",
                                                            "n_p2p", "p2p_pairs")},
            "clocks": clk}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    # FMM_BENCH_DIST=1 runs the distributed handle (NCCL) even at N=1 (a 1-rank communicator)
    use_dist = world > 1 or os.environ.get("FMM_BENCH_DIST") == "1"
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank,
                                world_size=world)
    xyz, q, n_all, cfg, scaling, desc = workload(args.config, world, rank)
    n_local = len(q)
    p = cfg["p"]
    X = torch.from_numpy(xyz).cuda()
    Q = torch.from_numpy(q).cuda()
    t0 = time.perf_counter()
    f = make_handle(cfg, args.mode, args.deterministic, distributed=use_dist)
    tune_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 512 MiB > L2

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        f.evaluate(X, Q)
    barrier()
    step_ms, phase, launches, clocks = time_steps(f, X, Q, args.steps, barrier, flush, stream, local)
    stats = f.stats()
    total_ms = sum(step_ms)
    t_max = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    total_ms = float(t_max.item())
    ms_step = total_ms / args.steps
    value = n_all / (ms_step * 1e-3)

    # end-to-end with host buffers: H2D of this step's inputs + evaluation + D2H of the results
    # inside the timed region (N=1: one fmm_evaluate_host C-ABI call; N>1: pinned copies around
    # the distributed evaluate)
    hx = torch.from_numpy(xyz).pin_memory().numpy()
    hq = torch.from_numpy(q).pin_memory().numpy()
    hphi = torch.empty(n_local, dtype=torch.float32).pin_memory().numpy()
    hgrad = torch.empty((n_local, 3), dtype=torch.float32).pin_memory().numpy()

    def e2e_step():
        if not use_dist:
            f.evaluate_host(hx, hq, hphi, hgrad)
        else:
            xd = torch.from_numpy(hx).to("cuda", non_blocking=True)
            qd = torch.from_numpy(hq).to("cuda", non_blocking=True)
            ph, gr = f.evaluate(xd, qd)
            torch.from_numpy(hphi).copy_(ph)
            torch.from_numpy(hgrad).copy_(gr)

    e2e_step()
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 5))):
        flush.fill_(1.0)
        barrier()
        t = time.perf_counter()
        e2e_step()
        torch.cuda.synchronize()
        e2e_ms.append(1e3 * (time.perf_counter() - t))
    e2e_t = torch.tensor([sum(e2e_ms) / len(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = n_all / (float(e2e_t.item()) * 1e-3)

    # the bit-reproducible mode (fmm_set_deterministic(1)): same workload, timed too
    det = None
    if not args.deterministic and not args.no_extras:
        fd = make_handle(cfg, args.mode, True, distributed=use_dist)
        try:
            for _ in range(args.warmup):
                fd.evaluate(X, Q)
            barrier()
            dms, dph, _, dclk = time_steps(fd, X, Q, max(3, min(args.steps, 10)), barrier, flush,
                                           stream, local)
        finally:
            fd.close()
        dt = torch.tensor([sum(dms) / len(dms)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        det = {"ms_per_step": float(dt.item()), "value": n_all / (float(dt.item()) * 1e-3),
               "unit": UNIT, "ms_m2l": dph["ms_m2l"], "phases_ms": dph, "clocks": dclk,
               "m2l_sum": "per-pair rows summed per target in list order (fmm_set_deterministic(1))"}

    # roofline: the dominant kernel of the step
    steps = args.steps
    m2l_ms = phase["ms_m2l"]
    # the P2P kernel alone (ms_p2p also covers its per-leaf descriptor and range-merge passes)
    p2p_ms = phase["ms_p2p_kernel"] or phase["ms_p2p"]
    m2l_gflops = stats["n_m2l"] * m2l_flops(p) / (m2l_ms * 1e-3) / 1e9 if m2l_ms > 0 else 0.0
    p2p_gflops = stats["p2p_pairs"] * P2P_FLOP_PER_PAIR / (p2p_ms * 1e-3) / 1e9 if p2p_ms > 0 else 0.0
    peak_gflops = N_SM * FP32_LANES_PER_SM * 2 * 1.965  # GFLOP/s at clocks.max.sm (B200_PROFILING)
    # M2L runs on the tcgen05 tensor cores (3xTF32) for p <= 10: its roofline is the TF32 tensor
    # peak = measured bf16 burst (MEASURED_PEAKS.json) x nominal tf32/bf16 ratio (1.1/2.25 PF)
    tc_dim = ((p + 1) ** 2 + 31) // 32 * 32
    m2l_tc_flops = 3 * 2 * tc_dim * tc_dim  # three TF32 MMAs per pair (hi.hi, hi.lo, lo.hi)
    try:
        bf16 = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
        tf32_src = "MEASURED_PEAKS.json bf16_tflops x 1.1/2.25 (nominal tf32/bf16), of measured"
    except (OSError, ValueError, KeyError):
        bf16, tf32_src = 1590.0, "B200_PROFILING fallback 1.59 PF bf16 x 1.1/2.25, of fallback"
    tf32_peak = bf16 * 1.1 / 2.25
    m2l_tensor_tflops = stats["n_m2l"] * m2l_tc_flops / (m2l_ms * 1e-3) / 1e12 if m2l_ms > 0 else 0.0
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    tkey = "" if args.config == "C2" else "_" + args.config
    p2p_line = {"bound": "alu", "kernel": "k_p2p_tma", "achieved": p2p_gflops / 1e3,
                "peak": peak_gflops / 1e3, "unit": "TFLOP/s", "frac": p2p_gflops / peak_gflops,
                "traffic": traffic.get("k_p2p_tma" + tkey),
                "peak_source": "148 SM x 128 FP32 lanes x 2 x 1.965 GHz (B200_PROFILING unit counts x "
                               "max clock); tools/peak_fp32 measured 74.0 TFLOP/s FFMA2",
                "flop_per_pair": P2P_FLOP_PER_PAIR}
    m2l_line = {"bound": "tensor", "kernel": "k_m2l_tc", "achieved": m2l_tensor_tflops,
                "peak": tf32_peak, "unit": "TFLOP/s", "frac": m2l_tensor_tflops / tf32_peak,
                "traffic": traffic.get("k_m2l_tc" + tkey), "peak_source": tf32_src,
                "tf32_flop_per_pair": m2l_tc_flops, "fp32_equiv_tflops": m2l_gflops / 1e3,
                "fp32_equiv_flop_per_pair": m2l_flops(p),
                "note": "time = the tcgen05 class GEMM launch, which also adds every pair's result into its target (red.global.add.v4.f32)"}
    if p2p_ms >= m2l_ms:
        roofline = dict(p2p_line, secondary=m2l_line)
    else:
        roofline = dict(m2l_line, secondary=p2p_line)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": desc, "n_total": n_all, "n_per_rank": n_local, "p": p,
                   "theta": cfg["theta"], "ncrit": cfg["ncrit"], "mode": args.mode,
                   "m2l_sum": ("ordered per-target reduction (fmm_set_deterministic(1))" if args.deterministic
                               else "L2 vector reductions, unordered (fmm_set_deterministic(0))"),
                   "l2": "inputs (16 B/particle) exceed L2 at C4; also flushed (512 MiB write) before every timed step"},
        "time_to_solution_ms": ms_step,
        "phases_ms": phase,
        "counts": {k: stats[k] for k in ("ncells", "nleaves", "depth", "n_m2l", "n_m2p", "n_p2p",
                                          "p2p_pairs", "m2p_evals")},
        "cost_model": dict(zip(("t_pp", "t_mp", "t_ml"), f.cost_model())),
        # SURVEY §8(d) interaction rates: kernel-only P2P pairs/s and M2L translations/s, and the
        # direct-sum-equivalent N(N-1)/T of the whole evaluation
        "interactions": {
            "p2p_pairs_per_s": stats["p2p_pairs"] / (p2p_ms * 1e-3) if p2p_ms > 0 else None,
            "m2l_per_s": stats["n_m2l"] / (m2l_ms * 1e-3) if m2l_ms > 0 else None,
            "effective_pairs_per_s": float(n_all) * (n_all - 1) / (ms_step * 1e-3)},
        "tune_s": tune_s,
        "gpu_launches": int(round(launches)) * steps,
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 16 * n_local,
                "d2h_bytes_per_step": 16 * n_local},
        "clocks": clocks,
    }
    if det is not None:
        line["deterministic"] = det
    if use_dist:
        line["comm"] = {k: stats[k] for k in ("n_global", "rank_lo", "rank_hi", "n_straddle",
                                               "let_cells", "let_particles", "bytes_sent", "ms_comm")}
        line["config"]["parallelism"] = f"Morton domain decomposition x{world}, LET alltoallv (NCCL)"
    f.close()
    if rank == 0 and world == 1 and not args.no_extras:
        line["other_configs"] = {
            name: extra_config(name, args.mode, max(3, min(args.steps, 20)), args.warmup, flush,
                               stream, local) for name in ("C2", "C3")}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(tuple(line["cost_model"].values()), cfg, args.mode)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=["C2", "C3", "C4", "C5"])
    ap.add_argument("--mode", default="hybrid", choices=["hybrid", "fmm", "treecode"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the C2/C3 and deterministic-mode extras")
    ap.add_argument("--dry-run", action="store_true", help="launch check only (no FMM)")
    ap.add_argument("--deterministic", action="store_true",
                    help="time the ordered M2L reduction (the library default) as the headline")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if world_size() > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines: the driver counts ranks
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


def world_size():
    return env_int("WORLD_SIZE", 1)


if __name__ == "__main__":
    main()
