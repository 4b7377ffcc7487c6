"""Synthetic inputs.  numpy.random.default_rng(seed) everywhere.

* bimodal(n, seed): p=0.8 U{32..256}, else U{4096..16384}  (80/20 mix, P:423-425,
  S:56; long range from the north_star).
* heavy(n, seed):   p=0.8 clip(round(exp(N(ln 128, 0.6))), 32, 2047),
                    else clip(floor(2048 * U^(-1/1.5)), 2048, 32768)  (Pareto 1.5 tail).
* arrivals: sorted Uniform(0, 600) s in fp32 -- Poisson arrivals conditioned on
  the count over one 600 s strategic window; pool index = arrival rank.
* cost_estimates: a per-request prefill-time *estimate* as an external
  predictor would supply it (the north_star's "estimated cost" field): the
  SPEC calibration curve times a lognormal(0, 0.1) predictor error.
  It is an opaque input to both the oracle and the CUDA path.
"""
from __future__ import annotations

import numpy as np

NOW = 600.0
DEFAULT_COST = (0.005, 0.0002, 1e-8)   # S:244 calibration, seconds
# Θ0: urgency in short queues, fairness in long ones
THETA0 = dict(a_b=0.0, b_b=1.0, a_u=-1e-4, b_u=2.0, a_f=1e-4, b_f=0.5)


def bimodal(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    short = rng.random(n) < 0.8
    s = rng.integers(32, 257, size=n)
    l = rng.integers(4096, 16385, size=n)
    return np.where(short, s, l).astype(np.int32)


def heavy(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    short = rng.random(n) < 0.8
    s = np.clip(np.rint(np.exp(rng.normal(np.log(128.0), 0.6, size=n))), 32, 2047)
    u = rng.random(n)
    u = np.where(u <= 0.0, np.finfo(np.float64).tiny, u)
    l = np.clip(np.floor(2048.0 * u ** (-1.0 / 1.5)), 2048, 32768)
    return np.where(short, s, l).astype(np.int32)


def lengths(kind: str, n: int, seed: int) -> np.ndarray:
    if kind == "bimodal":
        return bimodal(n, seed)
    if kind == "heavy":
        return heavy(n, seed)
    raise ValueError(kind)


def arrivals(n: int, seed: int, window: float = NOW, shuffled: bool = False) -> np.ndarray:
    rng = np.random.default_rng(seed + 7919)
    a = np.sort(rng.random(n) * window).astype(np.float32)
    if shuffled:
        rng.shuffle(a)
    return a


def cost_estimates(lens: np.ndarray, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed + 104729)
    b = lens.astype(np.float64)
    c0, c1, c2 = DEFAULT_COST
    base = c0 + c1 * b + c2 * b * b
    return (base * np.exp(rng.normal(0.0, 0.1, size=len(b)))).astype(np.float32)


def pool(kind: str, n: int, seed: int, shuffled: bool = False, with_cost: bool = True) -> dict:
    """A pending pool in structure-of-arrays form (len int32, arrival fp32, cost fp32)."""
    ln = lengths(kind, n, seed)
    out = {"len": ln, "arrival": arrivals(n, seed, shuffled=shuffled)}
    out["cost"] = cost_estimates(ln, seed) if with_cost else None
    return out


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rank r owns [floor(r n / P), floor((r+1) n / P)) of the pool."""
    return (rank * n) // world, ((rank + 1) * n) // world


def random_thetas(n_theta: int, seed: int) -> list[dict]:
    """C5: Θ uniform in S:500's bounds, a in [-0.01, 0.01], b in [0, 5]."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_theta):
        a = rng.uniform(-0.01, 0.01, size=3)
        b = rng.uniform(0.0, 5.0, size=3)
        out.append(dict(a_b=a[0], b_b=b[0], a_u=a[1], b_u=b[1], a_f=a[2], b_f=b[2]))
    return out


def quantile_bounds(history: np.ndarray, nq: int) -> list[tuple[int, int]]:
    """A balanced nq-quantile contiguous partition of a history (an alternative
    *input* partition for benchmarks); not the method."""
    h = np.sort(history.astype(np.int64))
    cuts = [int(h[0])]
    for i in range(1, nq):
        c = int(h[(i * len(h)) // nq])
        if c > cuts[-1]:
            cuts.append(c)
    top = int(h[-1]) + 1
    bounds = [(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)] + [(cuts[-1], top)]
    return bounds
