"""Seeded synthetic particle sets — the ONE module shared by the oracle side and the CUDA side.

It holds no arithmetic of the method (no keys, no tree, no expansions): it only draws
positions and charges. Both `oracle/` (through the tests) and the CUDA path (through the
tests and `bench.py`) receive the exact same float32 arrays from here.

Generator: NumPy's counter-based Philox4x32-10 bit generator, key = seed. Workloads follow
BASELINE.json's configs:

* ``uniform``  — x uniform in [0,1)^3, q = 1/N (PAPER.md:168 uses a random cube; SURVEY §8(c)
  reading 11 maps [-1,1]^3 to the unit cube of BASELINE.json).
* ``plummer``  — Plummer sphere, scale a = 1, q = 1/N, mass fraction X in (0, 0.999],
  r = a / sqrt(X^(-2/3) - 1), isotropic direction (Aarseth-Henon-Wielen sampling; BASELINE config 3).
* ``mixed``    — uniform positions, charges U(-1,1)/N (extra accuracy case, SURVEY §8(c) reading 10).
* ``shell``    — uniform on the unit sphere surface (PAPER.md:185 spherical shell), q = 1/N.

Seeds: C1 -> 1, C2 -> 2, C3 -> 3, C4 -> 4, C5 -> 5 + rank.
"""
from __future__ import annotations

import numpy as np

DISTRIBUTIONS = ("uniform", "plummer", "mixed", "shell")


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=int(seed)))


def make_particles(n: int, dist: str = "uniform", seed: int = 0):
    """Return (xyz float32 [n,3] C-contiguous, q float32 [n])."""
    n = int(n)
    if n < 0:
        raise ValueError("n must be >= 0")
    rng = _rng(seed)
    if dist in ("uniform", "mixed"):
        xyz = rng.random((n, 3), dtype=np.float32)
        if dist == "uniform":
            q = np.full(n, 1.0 / max(n, 1), dtype=np.float32)
        else:
            q = ((rng.random(n, dtype=np.float32) * 2.0 - 1.0) / max(n, 1)).astype(np.float32)
    elif dist == "plummer":
        u = rng.random((n, 3), dtype=np.float64)
        X = (1.0 - u[:, 0]) * 0.999  # (0, 0.999]
        r = 1.0 / np.sqrt(X ** (-2.0 / 3.0) - 1.0)
        cost = 2.0 * u[:, 1] - 1.0
        sint = np.sqrt(np.maximum(0.0, 1.0 - cost * cost))
        ph = 2.0 * np.pi * u[:, 2]
        xyz = np.stack([r * sint * np.cos(ph), r * sint * np.sin(ph), r * cost], axis=1).astype(np.float32)
        q = np.full(n, 1.0 / max(n, 1), dtype=np.float32)
    elif dist == "shell":
        u = rng.random((n, 2), dtype=np.float64)
        cost = 2.0 * u[:, 0] - 1.0
        sint = np.sqrt(np.maximum(0.0, 1.0 - cost * cost))
        ph = 2.0 * np.pi * u[:, 1]
        xyz = np.stack([sint * np.cos(ph), sint * np.sin(ph), cost], axis=1).astype(np.float32)
        q = np.full(n, 1.0 / max(n, 1), dtype=np.float32)
    else:
        raise ValueError(f"unknown distribution {dist!r}; choose from {DISTRIBUTIONS}")
    return np.ascontiguousarray(xyz), np.ascontiguousarray(q)


# BASELINE.json configs (SURVEY.md §8 notation C1..C5)
CONFIGS = {
    "C1": dict(n=1000, dist="uniform", seed=1, p=4, theta=0.5, ncrit=16),
    "C2": dict(n=1_000_000, dist="uniform", seed=2, p=10, theta=0.4, ncrit=64),
    "C3": dict(n=4_000_000, dist="plummer", seed=3, p=10, theta=0.4, ncrit=64),
    "C4": dict(n=16_000_000, dist="uniform", seed=4, p=10, theta=0.4, ncrit=64),
    "C5": dict(n=8_000_000, dist="uniform", seed=5, p=10, theta=0.4, ncrit=64),  # per rank, seed 5+rank
}
