"""Pins of oracle O14 (exact 1-D k-means for any k, reading R32; the k-means-only
partitions of Table 3 "EWSJF (K-Means)") against things other
than itself: exhaustive search over every contiguous k-partition with exact
rational SSE (brute.kmeans_brute), O3's k<=3 optimum, SPEC's worked example
(S:131-133), the degenerate k = 1 / k >= distinct cases, and the partition
invariants (contiguity, coverage, each history value routes into its own
cluster's queue under R15's midpoint bounds)."""
import random
from fractions import Fraction as F

import numpy as np
import pytest

import oracle as O
from oracle import brute


def _sse(parts):
    tot = F(0)
    for p in parts:
        mu = F(sum(p), len(p))
        tot += sum((F(x) - mu) ** 2 for x in p)
    return tot


@pytest.mark.parametrize("seed", range(40))
def test_kmeans_dp_is_the_exact_optimum(seed):
    rng = random.Random(seed)
    n = rng.randint(1, 13)
    xs = [rng.randint(1, 40) for _ in range(n)]
    for k in range(1, 6):
        d = len(set(xs))
        parts = O.kmeans_dp(xs, k)
        assert len(parts) == min(k, d)
        assert sorted(sum(parts, [])) == sorted(xs)
        if k > d:
            continue
        best, args = brute.kmeans_brute(xs, k)
        assert _sse(parts) == best, (xs, k, parts)


def test_kmeans_dp_unique_optimum_cuts():
    # well separated groups: the optimum is unique and obvious
    xs = [5, 6, 7, 50, 52, 300, 301, 302, 303, 2000]
    assert O.kmeans_dp(xs, 4) == [[5, 6, 7], [50, 52], [300, 301, 302, 303], [2000]]
    assert O.kmeans_dp(xs, 2) == [[5, 6, 7, 50, 52, 300, 301, 302, 303], [2000]]


def test_kmeans_dp_spec_example_and_k3_value():
    # S:131-133 (k = 3), and for k <= 3 the DP optimum equals O3's optimum value
    xs = [1, 2, 3, 100, 101, 102, 1000, 1001]
    assert O.kmeans_dp(xs, 3) == [[1, 2, 3], [100, 101, 102], [1000, 1001]]
    rng = random.Random(7)
    for _ in range(30):
        ys = [rng.randint(1, 60) for _ in range(rng.randint(3, 14))]
        for k in (1, 2, 3):
            if k > len(set(ys)):
                continue
            assert _sse(O.kmeans_dp(ys, k)) == _sse(O.kmeans(ys, k))


def test_kmeans_dp_degenerate():
    xs = [4, 4, 9, 9, 9, 20]
    assert O.kmeans_dp(xs, 1) == [sorted(xs)]
    assert O.kmeans_dp(xs, 3) == [[4, 4], [9, 9, 9], [20]]       # k = distinct: one cluster per value
    assert O.kmeans_dp(xs, 7) == [[4, 4], [9, 9, 9], [20]]       # k > distinct -> k = distinct


@pytest.mark.parametrize("k", [5, 10, 30])
def test_partition_kmeans_invariants(k):
    import workload
    h = workload.bimodal(10_000, 101)
    s, part, st = O.partition_kmeans(h, k)
    assert s == O.OK and part.n == k == st.k_used
    qs = part.queues()
    assert qs[0]["min_len"] == h.min() and qs[-1]["max_len"] == h.max() + 1
    for a, b in zip(qs, qs[1:]):
        assert a["max_len"] == b["min_len"] and a["min_len"] < a["max_len"]
    assert sum(q["count"] for q in qs) == len(h)
    # every value lands in the queue of its own cluster (R15 midpoint ownership)
    parts = O.kmeans_dp(h, k)
    lo = np.array([q["min_len"] for q in qs])
    for i, p in enumerate(parts):
        idx = np.searchsorted(lo, np.array(p), side="right") - 1
        assert (idx == i).all()
        assert qs[i]["count"] == len(p) and qs[i]["sum"] == sum(p)
