#!/usr/bin/env python
"""bench.py — FMM time-to-solution on B200 (BASELINE.json metric), driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload at N=1: BASELINE.json configs[1] = C2, N = 1,000,000 uniform random charges in the unit
cube, Laplace potential + gradient, p = 10, theta = 0.4, ncrit = 64, hybrid M2L/M2P/P2P choice
auto-tuned on the device. One step = one full fmm_evaluate (tree build, upward
sweep, traversal, M2L/M2P/P2P, downward sweep) on inputs already resident in HBM; L2 is flushed
(a 512 MiB write) before every timed step, outside the timed interval. `value` = particles
evaluated per second over all ranks (N / time-to-solution); `ms_per_step` = time-to-solution.

N > 1 (torchrun, one process per GPU): one distributed handle per rank (fmm_create_dist, NCCL
inside libfmm.so); weak scaling, each rank contributes one C2 instance shifted into
its own unit cube, so the job is ONE global problem of N x 1M particles; rank 0 prints.

`--impl reference` times the CPU FP64 oracle (oracle/, the only other arm this tier has) on the
host cores: each step is the full oracle FMM of a bounded instance of the same recipe.
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
P2P_FLOP_PER_PAIR = 18      # 3 FADD d, 1 FMUL + 2 FFMA r^2, 2 FMUL q/r^3, 1 FMUL q/r, 1 FADD, 3 FFMA
CPU_SAMPLE_N = 1_000_000  # cpu_baseline: the full C2 instance (about 6-10 s of the FP64 oracle)
REF_SAMPLE_N = 125_000    # --impl reference steps: C2 recipe at 1/8 size (same leaf occupancy)


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


def cpu_baseline(cost, p, theta, ncrit, mode_name):
    """The FP64 oracle as it stands, on this host's cores (rank 0, N=1 only)."""
    from oracle import oracle as O

    xyz, q = make_particles(CPU_SAMPLE_N, "uniform", 2)
    mode = {"hybrid": O.HYBRID, "fmm": O.FMM, "treecode": O.TREECODE}[mode_name]
    t = time.perf_counter()
    O.fmm(xyz, q, p, theta, ncrit, mode, cost=cost, want_structure=False)
    dt = time.perf_counter() - t
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": CPU_SAMPLE_N / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "seconds": dt, "single_thread": single_thread_oracle(cost),
            "sample": f"full oracle FMM (FP64, OpenMP) of the {CPU_SAMPLE_N}-particle C2 instance "
                      f"(same seed as the GPU workload (uniform cube, q=1/N, p={p}, theta={theta}, ncrit={ncrit}, "
                      f"{mode_name}, the GPU's measured cost model)"}


def single_thread_oracle(cost):
    """the oracle also on ONE thread (OMP_NUM_THREADS=1, a subprocess): C1 in full
    and a 62,500-particle instance of the C2 recipe (1/16 of C2, same leaf occupancy)."""
    code = (
        "import sys, time, json; sys.path.insert(0, %r)\n"
        "from fmm_inputs import CONFIGS, make_particles\n"
        "from oracle import oracle as O\n"
        "out = {}\n"
        "c = CONFIGS['C1']; x, q = make_particles(c['n'], c['dist'], c['seed'])\n"
        "t = time.perf_counter(); O.fmm(x, q, c['p'], c['theta'], c['ncrit'], O.HYBRID, cost=%r, want_structure=False)\n"
        "out['C1'] = c['n'] / (time.perf_counter() - t)\n"
        "x, q = make_particles(62500, 'uniform', 2)\n"
        "t = time.perf_counter(); O.fmm(x, q, 10, 0.4, 64, O.HYBRID, cost=%r, want_structure=False)\n"
        "out['C2_sample_62500'] = 62500 / (time.perf_counter() - t)\n"
        "print(json.dumps(out))\n") % (ROOT, tuple(cost), tuple(cost))
    env = dict(os.environ, OMP_NUM_THREADS="1")
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                           timeout=120)
        vals = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 -- a reporting extra; never fail the bench on it
        return {"error": str(e)[:200]}
    return {"cores": 1, "unit": UNIT, "C1_particles_per_s": vals["C1"],
            "C2_recipe_62500_particles_per_s": vals["C2_sample_62500"]}


def run_reference(args):
    """--impl reference: the CPU oracle arm (rank 0 only)."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    from oracle import oracle as O

    cfg = CONFIGS["C2"]
    xyz, q = make_particles(REF_SAMPLE_N, "uniform", 2)
    cost = (1.3e-12, 4.1e-10, 7.7e-9)  # a B200 cost model (measured by fmm_create), fixed here
    times = []
    for it in range(args.warmup + args.steps):
        t = time.perf_counter()
        O.fmm(xyz, q, cfg["p"], cfg["theta"], cfg["ncrit"], O.HYBRID, cost=cost, want_structure=False)
        if it >= args.warmup:
            times.append(time.perf_counter() - t)
    ms = 1e3 * sum(times) / len(times)
    value = REF_SAMPLE_N / (ms * 1e-3)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C2 recipe, bounded instance N={REF_SAMPLE_N}", "n": REF_SAMPLE_N,
                   "p": cfg["p"], "theta": cfg["theta"], "ncrit": cfg["ncrit"], "mode": "hybrid"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"each step: full FP64 oracle FMM of a {REF_SAMPLE_N}-particle "
                                   "instance of the C2 recipe on the host cores"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1108_5815_b200 import FMM

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    # FMM_BENCH_DIST=1 runs the distributed handle (NCCL) even at N=1 (a 1-rank communicator)
    use_dist = world > 1 or os.environ.get("FMM_BENCH_DIST") == "1"
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank,
                                world_size=world)
        from paper_1108_5815_b200.dist import DistFMM
    cfg = dict(CONFIGS[args.config])
    p, theta, ncrit = cfg["p"], cfg["theta"], cfg["ncrit"]
    if world == 1:
        n_local = cfg["n"]
        xyz, q = make_particles(n_local, cfg["dist"], cfg["seed"])
    else:  # weak scaling: C2 per rank, seeds 2 + rank, one global problem of world * 1M
        n_local = cfg["n"]
        xyz, q = make_particles(n_local, cfg["dist"], cfg["seed"] + 100 * rank)
        xyz = (xyz + np.array([rank % 2, (rank // 2) % 2, rank // 4], np.float32)).astype(np.float32)
    X = torch.from_numpy(xyz).cuda()
    Q = torch.from_numpy(q).cuda()
    t0 = time.perf_counter()
    if use_dist:  # distributed handle: NCCL communicator inside libfmm (fmm_create_dist)
        f = DistFMM(p=p, theta=theta, ncrit=ncrit, mode=args.mode, tune=args.deterministic)
    else:
        f = FMM(p=p, theta=theta, ncrit=ncrit, mode=args.mode, tune=args.deterministic)
    f.set_deterministic(args.deterministic)
    if not args.deterministic:
        f.tune()  # the kernel pre-calculation times the M2L the evaluations will use
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
    f.set_timing(True)
    step_ms, phase = [], {"ms_m2l": 0.0, "ms_p2p": 0.0, "ms_m2p": 0.0, "ms_tree": 0.0,
                          "ms_upward": 0.0, "ms_traverse": 0.0, "ms_downward": 0.0}
    launches = 0
    with ClockSampler(local) as clk:
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/": the launch list
        for _ in range(args.steps):
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
    stats = f.stats()
    total_ms = sum(step_ms)
    t_max = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    total_ms = float(t_max.item())
    ms_step = total_ms / args.steps
    n_all = n_local * world
    value = n_all / (ms_step * 1e-3)

    # end-to-end with host buffers: H2D of this step's inputs + evaluation + D2H of the results
    # inside the timed region (N=1: one fmm_evaluate_host C-ABI call; N>1: pinned copies around
    # the distributed evaluate)
    hx = torch.from_numpy(xyz).pin_memory().numpy()
    hq = torch.from_numpy(q).pin_memory().numpy()
    hphi = torch.empty(n_local, dtype=torch.float32).pin_memory().numpy()
    hgrad = torch.empty((n_local, 3), dtype=torch.float32).pin_memory().numpy()
    f.set_timing(False)

    def e2e_step():
        if world == 1:
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

    # roofline: the dominant kernel of the step, FP32 ALU bound (CUDA cores, not tensor cores)
    steps = args.steps
    m2l_ms = phase["ms_m2l"] / steps
    p2p_ms = phase["ms_p2p"] / steps
    m2l_gflops = stats["n_m2l"] * m2l_flops(p) / (m2l_ms * 1e-3) / 1e9 if m2l_ms > 0 else 0.0
    p2p_gflops = stats["p2p_pairs"] * P2P_FLOP_PER_PAIR / (p2p_ms * 1e-3) / 1e9 if p2p_ms > 0 else 0.0
    peak_gflops = N_SM * FP32_LANES_PER_SM * 2 * 1.965  # GFLOP/s at clocks.max.sm (B200_PROFILING)
    # M2L runs on the tcgen05 tensor cores (3xTF32) for p <= 10: its roofline is the TF32 tensor
    # peak = measured bf16 burst (MEASURED_PEAKS.json) x nominal tf32/bf16 ratio (1.1/2.25 PF)
    tc_dim = ((p + 1) ** 2 + 31) // 32 * 32
    m2l_tc_flops = 3 * 2 * tc_dim * tc_dim  # three TF32 MMAs per pair (hi.hi, hi.lo, lo.hi)
    try:
        bf16 = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
        tf32_src = "MEASURED_PEAKS.json bf16_tflops x 1.1/2.25 (nominal tf32/bf16)"
    except (OSError, ValueError, KeyError):
        bf16, tf32_src = 1590.0, "B200_PROFILING fallback 1.59 PF bf16 x 1.1/2.25"
    tf32_peak = bf16 * 1.1 / 2.25
    m2l_tensor_tflops = stats["n_m2l"] * m2l_tc_flops / (m2l_ms * 1e-3) / 1e12 if m2l_ms > 0 else 0.0
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    p2p_line = {"bound": "alu", "kernel": "k_p2p_leaves", "achieved": p2p_gflops / 1e3,
                "peak": peak_gflops / 1e3, "unit": "TFLOP/s", "frac": p2p_gflops / peak_gflops,
                "traffic": traffic.get("k_p2p_leaves"),
                "peak_source": "148 SM x 128 FP32 lanes x 2 x 1.965 GHz (B200_PROFILING unit counts x "
                               "max clock); tools/peak_fp32 measured 74.0 TFLOP/s FFMA2",
                "flop_per_pair": P2P_FLOP_PER_PAIR}
    m2l_line = {"bound": "tensor", "kernel": "k_m2l_tc", "achieved": m2l_tensor_tflops,
                "peak": tf32_peak, "unit": "TFLOP/s", "frac": m2l_tensor_tflops / tf32_peak,
                "traffic": traffic.get("k_m2l_tc"), "peak_source": tf32_src,
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
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "C2: N=1M uniform cube, Laplace phi+grad, p=10, theta=0.4, ncrit=64, "
                               "auto-tuned hybrid" if world == 1 else
                               f"C2 per rank ({world} x 1M, one global problem)",
                   "n_per_rank": n_local, "p": p, "theta": theta, "ncrit": ncrit, "mode": args.mode,
                   "m2l_sum": ("ordered per-target reduction (fmm_set_deterministic(1))" if args.deterministic
                               else "L2 vector reductions, unordered (fmm_set_deterministic(0))"),
                   "l2": "flushed (512 MiB write) before every timed step"},
        "time_to_solution_ms": ms_step,
        "phases_ms": {k: v / steps for k, v in phase.items()},
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
        "gpu_launches": launches,
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 16 * n_local,
                "d2h_bytes_per_step": 16 * n_local},
        "clocks": clk.summary(),
    }
    if use_dist:
        line["comm"] = {k: stats[k] for k in ("n_global", "rank_lo", "rank_hi", "n_straddle",
                                               "let_cells", "let_particles", "bytes_sent", "ms_comm")}
        line["config"]["parallelism"] = f"Morton domain decomposition x{world}, LET alltoallv (NCCL)"
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(f.cost_model(), p, theta, ncrit, args.mode)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--mode", default="hybrid", choices=["hybrid", "fmm", "treecode"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--deterministic", action="store_true",
                    help="ordered M2L reduction (the library default); default here: L2 reductions")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
