"""Exact brute-force references (fractions.Fraction) for tiny inputs — TEST ONLY.

These are written independently of ewsjf_oracle.c, straight from the paper's
definitions in exact rational arithmetic, to PIN the oracle:

* kmeans_brute      — every contiguous k-partition of the sorted multiset, exact
                      SSE ("exhaustive search over all contiguous 3-partitions").
* refine_brute      — Eq. 2 with mean(G) taken literally as the arithmetic mean
                      of the gap list G, no telescoping shortcut.
* prune_brute       — Eq. 3 with exact densities/means.
* bubble_brute      — Alg. 2 line by line with the real multipliers 11/10, 9/10
                      and real range/2, then the covered integer lengths.
* topk_brute        — the K-subset whose every member beats every non-member,
                      by enumerating subsets (north_star "brute-force optimal
                      selection ... on pools of 20 requests or fewer").
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction as F


def _sse(xs):
    n = len(xs)
    mu = F(sum(xs), n)
    return sum((F(x) - mu) ** 2 for x in xs)


def kmeans_brute(values, k):
    """Return (min_sse, [optimal partitions]) over contiguous k-partitions of sorted(values)."""
    xs = sorted(values)
    n = len(xs)
    best, arg = None, []
    for cuts in itertools.combinations(range(1, n), k - 1):
        b = (0,) + cuts + (n,)
        parts = [xs[b[i]:b[i + 1]] for i in range(k)]
        s = sum(_sse(p) for p in parts)
        if best is None or s < best:
            best, arg = s, [parts]
        elif s == best:
            arg.append(parts)
    return best, arg


def refine_brute(values, alpha, min_width=1):
    """SPEC refine_cluster with G as an explicit list (multiset gaps)."""
    xs = sorted(values)
    a = F(alpha)
    if len(xs) < 2:
        return [xs]
    span = xs[-1] - xs[0]
    if span == 0 or span < min_width:
        return [xs]
    G = [xs[i + 1] - xs[i] for i in range(len(xs) - 1)]
    meanG = F(sum(G), len(G))
    cut = [i for i, g in enumerate(G) if F(g) > a * meanG]
    if not cut:
        return [xs]
    out, s = [], 0
    for i in cut:
        out += refine_brute(xs[s:i + 1], alpha, min_width)
        s = i + 1
    out += refine_brute(xs[s:], alpha, min_width)
    return out


def prune_brute(queues, max_queues, eps, rule="min"):
    """queues = [(lo, hi, [members...]), ...]; merge per Eq. 3 until <= max_queues."""
    qs = [(lo, hi, list(m)) for lo, hi, m in queues]
    e = F(eps)
    while len(qs) > max_queues and len(qs) > 1:
        us = []
        for p in range(len(qs) - 1):
            (l1, h1, m1), (l2, h2, m2) = qs[p], qs[p + 1]
            r1, r2 = F(len(m1), h1 - l1), F(len(m2), h2 - l2)
            mu1, mu2 = F(sum(m1), len(m1)), F(sum(m2), len(m2))
            us.append((r1 + r2) / (abs(mu2 - mu1) + e))
        target = min(us) if rule == "min" else max(us)
        p = us.index(target)
        (l1, h1, m1), (l2, h2, m2) = qs[p], qs[p + 1]
        qs[p:p + 2] = [(l1, h2, m1 + m2)]
    return qs


def bubble_brute(L, left_max, right_min, bubble_width):
    """Alg. 2 for one gap-falling L between Q_i.max_len and Q_{i+1}.min_len.
    Returns 'left', 'right' or the new integer interval (lo, hi)."""
    if L <= F(left_max) * F(11, 10):
        return "left"
    if L >= F(right_min) * F(9, 10):
        return "right"
    available = right_min - left_max
    rng = min(bubble_width, available)
    new_min = max(F(L) - F(rng, 2), F(left_max))
    new_max = min(F(L) + F(rng, 2), F(right_min))
    # the integer lengths covered by the real interval [new_min, new_max)
    return (math.ceil(new_min), math.ceil(new_max))


def topk_brute(keys, K):
    """keys: list of comparable keys (larger = better); returns the index set of
    the unique K-subset whose members all beat all non-members."""
    n = len(keys)
    K = min(K, n)
    found = []
    for S in itertools.combinations(range(n), K):
        inside = set(S)
        lo = min((keys[i] for i in S), default=None)
        hi = max((keys[i] for i in range(n) if i not in inside), default=None)
        if hi is None or lo is None or lo > hi:
            found.append(inside)
    assert len(found) == 1
    return found[0]


def score_exact(index, b, W, C, w_base, w_urg, w_fair, log_term=None):
    """Eq. 4 with exact rationals except the log term."""
    lt = F(math.log(b + 1)) if log_term is None else F(log_term)
    qf = F(index) / (F(b) + 1)
    return qf * (F(w_base) + F(w_urg) * F(W) / F(C) + F(w_fair) * lt)
