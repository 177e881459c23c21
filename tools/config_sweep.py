"""Time-to-solution / interaction rates of the BASELINE configs beyond the bench line (SURVEY
§8(d): C3 Plummer, C4 16M and C5's 8M per-GPU slice on one B200; the evaluation modes (E8); the
p ladder (E11); the theta x ncrit sweep of C5 (E6/E10)). One JSON line per run on stdout.

Timing: CUDA events around fmm_evaluate on resident inputs, L2 flushed before every step, median
of `--steps` after 3 warm-ups, the handle auto-tuned on the device; every line carries the
nvidia-smi clock record of its timed steps (bench.ClockSampler). Accuracy in the sweep is measured
against the FP64 oracle's direct sum (oracle.direct, test infrastructure) on 2,048 sampled
particles.
Also the paper's own GPU experiments as B200 analogs: E7 interaction mix on a spherical
shell, E10 time vs N of treecode / FMM / hybrid at N_crit = 100, p = 8.
Usage: config_sweep.py [configs|modes|pladder|sweep|mix|nsweep|paper|all] [--steps K]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import ClockSampler  # noqa: E402
from fmm_inputs import CONFIGS, make_particles
from paper_1108_5815_b200 import FMM

P2P_FLOP = 19
LAST_CLOCKS = {}


def m2l_flop(p):
    return 2 * (p + 1) ** 4


def timed(f, X, Q, steps, flush):
    for _ in range(3):
        f.evaluate(X, Q)
    f.set_timing(True)
    ms, st = [], []
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            phi, grad = f.evaluate(X, Q)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            st.append(f.stats())
    LAST_CLOCKS.clear()
    LAST_CLOCKS.update(clk.summary())
    f.set_timing(False)
    i = int(np.argsort(ms)[len(ms) // 2])
    return ms[i], st[i], phi, grad


def record(tag, cfg, n, mode, p, theta, ncrit, ms, s, f, extra=None):
    line = {"run": tag, "config": cfg, "n": n, "mode": mode, "p": p, "theta": theta,
            "ncrit": ncrit, "time_to_solution_ms": round(ms, 4),
            "particles_per_s": n / (ms * 1e-3),
            "phases_ms": {k: round(s[k], 4) for k in ("ms_tree", "ms_upward", "ms_traverse", "ms_m2l",
                                                        "ms_p2p", "ms_m2p", "ms_downward")},
            "counts": {k: s[k] for k in ("ncells", "nleaves", "depth", "n_m2l", "n_m2p", "n_p2p",
                                          "p2p_pairs", "m2p_evals")},
            "p2p_pairs_per_s": s["p2p_pairs"] / (s["ms_p2p"] * 1e-3) if s["ms_p2p"] > 0 else None,
            "p2p_tflops": P2P_FLOP * s["p2p_pairs"] / (s["ms_p2p"] * 1e-3) / 1e12 if s["ms_p2p"] > 0 else None,
            "m2l_per_s": s["n_m2l"] / (s["ms_m2l"] * 1e-3) if s["ms_m2l"] > 0 else None,
            "m2l_fp32equiv_tflops": m2l_flop(p) * s["n_m2l"] / (s["ms_m2l"] * 1e-3) / 1e12 if s["ms_m2l"] > 0 else None,
            "cost_model": dict(zip(("t_pp", "t_mp", "t_ml"), f.cost_model())),
            "clocks": dict(LAST_CLOCKS)}
    if extra:
        line.update(extra)
    print(json.dumps(line), flush=True)
    return line


def rel_l2(a, b):
    return float(torch.linalg.norm((a - b).double()) / torch.linalg.norm(b.double()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="?", default="all")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
    what = a.what

    def run_cfg(name, mode="hybrid", p=None, theta=None, ncrit=None, n=None, extra=None):
        c = CONFIGS[name]
        p, theta, ncrit, n = p or c["p"], theta or c["theta"], ncrit or c["ncrit"], n or c["n"]
        xyz, q = make_particles(n, c["dist"], c["seed"])
        X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
        f = FMM(p=p, theta=theta, ncrit=ncrit, mode=mode, tune=False)
        f.set_deterministic(False)
        f.tune()
        ms, s, phi, grad = timed(f, X, Q, a.steps, flush)
        line = record(name, name, n, mode, p, theta, ncrit, ms, s, f, extra)
        f.close()
        return line, X, Q, phi, grad

    if what in ("configs", "all"):
        for name in ("C2", "C3", "C5", "C4"):
            run_cfg(name)
    if what in ("modes", "all"):
        for mode in ("fmm", "treecode"):
            run_cfg("C2", mode=mode)
    if what in ("pladder", "all"):
        for p in (4, 6, 8, 12):
            run_cfg("C2", p=p)
    if what in ("mix", "paper", "all"):
        # E7: spherical shell, N = 1e5, N_crit = 20: interaction mix per mode
        xyz, q = make_particles(100_000, "shell", 7)
        X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
        for mode in ("treecode", "fmm", "hybrid"):
            f = FMM(p=10, theta=0.4, ncrit=20, mode=mode, tune=False)
            f.set_deterministic(False)
            f.tune()
            ms, s, _, _ = timed(f, X, Q, a.steps, flush)
            c = s
            record("E7-shell-mix", "shell", 100_000, mode, 10, 0.4, 20, ms, s, f,
                   {"mix": {"m2p_per_p2p": c["n_m2p"] / max(1, c["n_p2p"]),
                            "m2l_per_p2p": c["n_m2l"] / max(1, c["n_p2p"]),
                            "p2p_per_m2l": c["n_p2p"] / max(1, c["n_m2l"])}})
            f.close()
    if what in ("nsweep", "paper", "all"):
        # E10: time vs N of the three methods at N_crit = 100, p = 8, uniform cube
        for n in (100_000, 300_000, 1_000_000, 3_000_000, 10_000_000):
            xyz, q = make_particles(n, "uniform", 10)
            X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
            for mode in ("treecode", "fmm", "hybrid"):
                if mode == "treecode" and n > 3_000_000:
                    continue
                f = FMM(p=8, theta=0.4, ncrit=100, mode=mode, tune=False)
                f.set_deterministic(False)
                f.tune()
                ms, s, _, _ = timed(f, X, Q, max(3, a.steps // 2), flush)
                record("E10-nsweep", "uniform", n, mode, 8, 0.4, 100, ms, s, f)
                f.close()
    if what in ("sweep", "all"):
        c = CONFIGS["C5"]
        xyz, q = make_particles(c["n"], c["dist"], c["seed"])
        X, Q = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
        from oracle import oracle as O  # test infrastructure: the reference direct sum only

        sample = np.random.default_rng(5).choice(c["n"], 2048, replace=False)
        dphi, dgrad = O.direct(xyz, q, sample)
        sidx = torch.from_numpy(sample).cuda()
        best = None
        for theta in (0.3, 0.4, 0.5):
            for ncrit in (16, 32, 64, 128, 256):
                f = FMM(p=10, theta=theta, ncrit=ncrit, mode="hybrid", tune=False)
                f.set_deterministic(False)
                f.tune()
                ms, s, phi, grad = timed(f, X, Q, max(3, a.steps // 2), flush)
                ph = phi[sidx].double().cpu().numpy()
                gr = grad[sidx].double().cpu().numpy()
                ep = float(np.linalg.norm(ph - dphi) / np.linalg.norm(dphi))
                eg = float(np.linalg.norm(gr - dgrad) / np.linalg.norm(dgrad))
                line = record("C5-sweep", "C5", c["n"], "hybrid", 10, theta, ncrit, ms, s, f,
                              {"err_phi_vs_direct": ep, "err_grad_vs_direct": eg})
                f.close()
                if ep < 1e-4 and (best is None or ms < best["time_to_solution_ms"]):
                    best = line
        print(json.dumps({"run": "C5-sweep-best", "theta": best["theta"], "ncrit": best["ncrit"],
                          "time_to_solution_ms": best["time_to_solution_ms"]}), flush=True)


if __name__ == "__main__":
    main()
