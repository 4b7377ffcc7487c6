"""Pin the CPU oracle to things other than itself (runs on CPU: -m "not gpu").

Pins: SPEC worked examples (tests/golden/spec_examples.json, each cited),
exact Fraction brute force (oracle/brute.py) on tiny inputs, closed forms,
library special cases (numpy searchsorted / lexsort / bincount) and the
invariants SPEC states.
"""
import json
import math
import os
from fractions import Fraction as Fr

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st, HealthCheck

from oracle import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------- Stage 1 (A3) ---
@pytest.mark.parametrize("ex", GOLD["kmeans"], ids=lambda e: e["cite"][:20])
def test_kmeans_golden(orc, ex):
    assert orc.kmeans(ex["values"], ex["k"]) == ex["expected"]


@settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.lists(st.integers(1, 60), min_size=3, max_size=14), st.integers(1, 3))
def test_kmeans_vs_exhaustive_fraction(orc, xs, k):
    """Oracle's cut attains the exact minimum SSE over ALL contiguous k-partitions
    (S:131 exhaustive search), and equals it when the optimum is unique."""
    k = min(k, len(set(xs)))
    got = orc.kmeans(xs, k)
    best, args = brute.kmeans_brute(xs, k)
    sse = sum(brute._sse(p) for p in got)
    assert sse == best
    if len(args) == 1:
        assert got == args[0]


def test_kmeans_invalid_k(orc):
    with pytest.raises(ValueError):
        orc.kmeans([1, 2], 3)


# ------------------------------------------------------------- Stage 2 (A4) ---
@pytest.mark.parametrize("ex", GOLD["refine"], ids=lambda e: e["cite"][:20])
def test_refine_golden(orc, ex):
    assert orc.refine(ex["values"], ex["alpha"], ex["min_width"]) == ex["expected"]


@settings(max_examples=300, deadline=None)
@given(st.lists(st.integers(1, 400), min_size=1, max_size=40),
       st.sampled_from([1.25, 1.5, 2.0, 2.5, 3.0, 4.0]), st.sampled_from([1, 2, 5, 50]))
def test_refine_vs_literal_eq2(orc, xs, alpha, mw):
    """Eq. 2 with mean(G) as the literal mean of the gap list (exact Fractions)
    reproduces the oracle's telescoped g*(n-1) > alpha*span test at every node
    (acceptance #5's per-node re-check).  Dyadic alpha keeps alpha*span exact."""
    assert orc.refine(xs, alpha, mw) == brute.refine_brute(xs, alpha, mw)


@settings(max_examples=200, deadline=None)
@given(st.lists(st.integers(1, 300), min_size=2, max_size=60))
def test_refine_concatenation_preserves_input(orc, xs):
    """refine output concatenated in order equals its input."""
    parts = orc.refine(xs, 2.0, 1)
    assert sum(parts, []) == sorted(xs)


# ------------------------------------------------------------- Stage 3 (A6) ---
@pytest.mark.parametrize("ex", GOLD["utility"], ids=lambda e: e["cite"][:20])
def test_utility_golden(orc, ex):
    got = orc.utility(ex["rho"][0], ex["rho"][1], ex["mean"][0], ex["mean"][1], ex["eps"])
    assert got == pytest.approx(ex["expected"], rel=1e-15, abs=0)


def _prune_args(queues):
    lo = [q[0] for q in queues]; hi = [q[1] for q in queues]
    cnt = [len(q[2]) for q in queues]; s1 = [sum(q[2]) for q in queues]; s2 = [sum(x * x for x in q[2]) for q in queues]
    return lo, hi, cnt, s1, s2


@pytest.mark.parametrize("ex", GOLD["prune"], ids=lambda e: e["cite"][:20])
def test_prune_golden(orc, ex):
    lo, hi, cnt, s1, s2 = _prune_args(ex["queues"])
    if "expected_u" in ex:   # the constructed utilities really are 0.5 and 2.0
        r = [c / (h - l) for l, h, c in zip(lo, hi, cnt)]
        mu = [a / c for a, c in zip(s1, cnt)]
        u = [orc.utility(r[i], r[i + 1], mu[i], mu[i + 1], ex["eps"]) for i in range(2)]
        assert u == pytest.approx(ex["expected_u"], rel=1e-12)
    L, H, *_ = orc.prune(lo, hi, cnt, s1, s2, ex["max_queues"], ex["eps"])
    assert [[int(a), int(b)] for a, b in zip(L, H)] == ex["expected_bounds"]


@settings(max_examples=200, deadline=None)
@given(st.lists(st.tuples(st.integers(1, 9), st.lists(st.integers(0, 8), min_size=1, max_size=6)),
                min_size=1, max_size=12),
       st.integers(1, 6), st.sampled_from(["min", "max"]))
def test_prune_vs_fraction_bruteforce(orc, spec, maxq, rule):
    """Merge sequence of Eq. 3 with exact rationals vs the fp64 oracle.
    Inputs are built so that the exact utilities have no near-ties."""
    queues, lo = [], 0
    for width, offs in spec:
        members = sorted(lo + (o % width) for o in offs)
        queues.append((lo, lo + width, members))
        lo += width
    # skip inputs with exact ties / near-ties in some iteration (fp64 may order them differently)
    eps = 2.0 ** -10
    ref = brute.prune_brute(queues, maxq, eps, rule)
    args = _prune_args(queues)
    L, H, cnt, s1, s2, merges = orc.prune(*args, maxq, eps, 0 if rule == "min" else 1)
    if not _no_near_ties(queues, maxq, eps, rule):
        return
    assert [(int(a), int(b)) for a, b in zip(L, H)] == [(q[0], q[1]) for q in ref]
    assert list(cnt) == [len(q[2]) for q in ref]
    assert merges == len(queues) - len(ref)


def _no_near_ties(queues, maxq, eps, rule):
    qs = [(lo, hi, list(m)) for lo, hi, m in queues]
    e = Fr(eps)
    while len(qs) > maxq and len(qs) > 1:
        us = []
        for p in range(len(qs) - 1):
            (l1, h1, m1), (l2, h2, m2) = qs[p], qs[p + 1]
            us.append((Fr(len(m1), h1 - l1) + Fr(len(m2), h2 - l2)) / (abs(Fr(sum(m2), len(m2)) - Fr(sum(m1), len(m1))) + e))
        s = sorted(us)
        if len(s) > 1:
            a, b = (s[0], s[1]) if rule == "min" else (s[-1], s[-2])
            if abs(a - b) <= abs(a) * Fr(1, 10 ** 9):
                return False
        t = min(us) if rule == "min" else max(us)
        p = us.index(t)
        (l1, h1, m1), (l2, h2, m2) = qs[p], qs[p + 1]
        qs[p:p + 2] = [(l1, h2, m1 + m2)]
    return True


# ------------------------------------------------------ R&P pipeline (A1-A6) ---
def _check_partition_invariants(orc, xs, part, maxq):
    qs = part.queues()
    assert 1 <= len(qs) <= maxq
    for a, b in zip(qs, qs[1:]):
        assert a["max_len"] == b["min_len"]                           # S:115 contiguity
    for q in qs:
        assert q["min_len"] < q["max_len"]
    assert [q["index"] for q in qs] == list(range(1, len(qs) + 1))
    v = np.asarray(xs)
    v = v[v >= 1]
    assert qs[0]["min_len"] == v.min() and qs[-1]["max_len"] == v.max() + 1   # coverage
    # every history value lands in exactly one queue, counts and sums match
    bounds = np.array([q["min_len"] for q in qs])
    pos = np.searchsorted(bounds, v, side="right") - 1
    assert (pos >= 0).all()
    cnt = np.bincount(pos, minlength=len(qs))
    s1 = np.zeros(len(qs), dtype=np.int64)
    s2 = np.zeros(len(qs), dtype=np.int64)
    np.add.at(s1, pos, v.astype(np.int64))
    np.add.at(s2, pos, v.astype(np.int64) ** 2)
    assert cnt.tolist() == [q["count"] for q in qs]
    assert s1.tolist() == [q["sum"] for q in qs]
    assert s2.tolist() == [q["sumsq"] for q in qs]                  # S2 = Σ b² (A2, P:285 mean/variance)
    # profile fields from first principles: b̄ = Σb/n, ρ = n/width (R16), SSE = Σ(b - b̄)²
    for i, q in enumerate(qs):
        mem = v[pos == i]
        assert q["mean"] == pytest.approx(float(Fr(int(mem.sum()), len(mem))), rel=1e-15)
        assert q["density"] == pytest.approx(len(mem) / (q["max_len"] - q["min_len"]), rel=1e-15)
        exact = sum((Fr(int(x)) - Fr(int(mem.sum()), len(mem))) ** 2 for x in mem)
        assert q["sse"] == pytest.approx(float(exact), rel=1e-9, abs=1e-6)


@settings(max_examples=200, deadline=None)
@given(st.lists(st.integers(1, 3000), min_size=1, max_size=300), st.integers(1, 12),
       st.sampled_from([1.5, 2.0, 3.0]))
def test_partition_invariants_random(orc, xs, maxq, alpha):
    """Acceptance #5: contiguity, disjointness, |Q| <= max_queues."""
    s, part, stt = orc.partition(xs, alpha=alpha, max_queues=maxq)
    assert s == orc.OK          # all lengths >= 1 here
    _check_partition_invariants(orc, xs, part, maxq)
    assert stt.segments - stt.merges == part.n


def test_partition_bimodal_split_in_gap(orc):
    """bimodal trace -> >= 2 queues with a boundary inside the empty gap.

    Holds under the MAX_U switch.  Under the literal MIN_U rule (R17, the default)
    Stage 3 degenerates as documented in DESIGN.md: 31 single-length queues
    [32,33)..[62,63) and one mega-queue [63, max+1) holding ~89% of the history
    (|Δb̄| in Eq. 3's denominator makes the growing merged queue the argmin)."""
    import workload
    xs = workload.bimodal(10000, 101)
    s, part, _ = orc.partition(xs, merge_rule=orc.MAX_U)
    qs = part.queues()
    assert s == orc.OK and len(qs) >= 2
    assert any(257 <= q["max_len"] <= 4096 for q in qs[:-1])
    _check_partition_invariants(orc, xs, part, 32)
    s, part, _ = orc.partition(xs)
    qs = part.queues()
    assert [(q["min_len"], q["max_len"]) for q in qs[:31]] == [(L, L + 1) for L in range(32, 63)]
    assert qs[31]["min_len"] == 63 and qs[31]["count"] / len(xs) > 0.85
    _check_partition_invariants(orc, xs, part, 32)


def test_partition_identical_lengths_one_queue(orc):
    s, part, _ = orc.partition([777] * 50)
    assert s == orc.OK and part.n == 1
    assert (part.q[0].min_len, part.q[0].max_len, part.q[0].count) == (777, 778, 50)


def test_partition_determinism_and_empty(orc):
    import workload
    xs = workload.heavy(20000, 5)
    a = orc.partition(xs)[1].queues()
    b = orc.partition(xs)[1].queues()
    assert a == b
    assert orc.partition([])[0] == orc.EMPTY
    assert orc.partition([0, -3])[0] == orc.EMPTY
    assert orc.partition([5, 6], alpha=1.0)[0] == orc.INVALID         # S:121 alpha > 1


def test_partition_stage_composition_small(orc):
    """R&P on tiny data == kmeans -> refine per cluster -> prune, via the brute references."""
    xs = [1, 2, 3, 5, 100, 101, 103, 180, 1000, 1001, 1003, 1500]
    s, part, st_ = orc.partition(xs, max_queues=3, epsilon=2.0 ** -10)
    _, args = brute.kmeans_brute(xs, 3)
    segs = []
    for c in args[0]:
        segs += brute.refine_brute(c, 2.0, 1)
    # midpoint finalization (R15)
    lo = [segs[0][0]]
    hi = []
    for i in range(len(segs) - 1):
        b = (segs[i][-1] + segs[i + 1][0]) // 2 + 1
        hi.append(b); lo.append(b)
    hi.append(segs[-1][-1] + 1)
    ref = brute.prune_brute(list(zip(lo, hi, segs)), 3, 2.0 ** -10)
    assert [(q["min_len"], q["max_len"]) for q in part.queues()] == [(a, b) for a, b, _ in ref]


# ------------------------------------------------------------ weights (A7) ---
@pytest.mark.parametrize("ex", GOLD["weights"], ids=lambda e: e["cite"][:20])
def test_weights_golden(orc, ex):
    w = orc.weights(orc.meta(**ex["theta"]), ex["mean"])
    which = {"S:309": 1, "S:310": 1, "S:311": 2}[ex["cite"][:5]]
    assert w[which] == pytest.approx(ex["expected"], abs=1e-7)


# -------------------------------------------------------- routing (A8, A9) ---
@pytest.mark.parametrize("ex", GOLD["route"], ids=lambda e: e["cite"][:20])
def test_route_golden(orc, ex):
    part = orc.make_partition(ex["bounds"])
    s, qid, *_ = orc.route([ex["b"]], part, 64)
    assert qid[0] == ex["expected_pos"]


@settings(max_examples=100, deadline=None)
@given(st.lists(st.integers(2, 50), min_size=1, max_size=20), st.lists(st.integers(-5, 1200), min_size=1, max_size=200))
def test_route_contiguous_is_searchsorted(orc, widths, lens):
    """On a contiguous partition routing reduces to searchsorted(min_len, b, 'right') - 1
    (SURVEY pins A8); nothing outside creates bubbles except off-range lengths."""
    edges = np.concatenate([[1], 1 + np.cumsum(widths)])
    bounds = list(zip(edges[:-1], edges[1:]))
    part = orc.make_partition(bounds)
    inside = [x for x in lens if 1 <= x < edges[-1]]
    s, qid, bad, made, dropped = orc.route(inside, part, 64)
    assert made == 0 and bad == 0
    np.testing.assert_array_equal(qid, np.searchsorted(edges[:-1], inside, side="right") - 1)


@pytest.mark.parametrize("ex", GOLD["bubble"], ids=lambda e: e["cite"][:20])
def test_bubble_golden(orc, ex):
    part = orc.make_partition([(1, ex["left_max"]), (ex["right_min"], 1000)])
    s, qid, bad, made, _ = orc.route([ex["L"]], part, ex["width"])
    qs = part.queues()
    if ex["expected"] == "left":
        assert qid[0] == 0 and made == 0
    elif ex["expected"] == "right":
        assert qid[0] == 1 and made == 0
    else:
        assert made == 1 and qs[1]["is_bubble"] == 1
        assert [qs[1]["min_len"], qs[1]["max_len"]] == ex["expected"]
        assert qid[0] == qs[1]["id"] == 2 and [q["index"] for q in qs] == [1, 2, 3]


@pytest.mark.parametrize("width", [40, 41, 1, 7, 100, 1000])
def test_bubble_exhaustive_sweep(orc, width):
    """Acceptance #6: every integer L in [100, 200] against the
    line-by-line exact-rational Alg. 2, fresh partition each time."""
    for L in range(100, 200):
        part = orc.make_partition([(1, 100), (200, 1000)])
        s, qid, bad, made, _ = orc.route([L], part, width)
        exp = brute.bubble_brute(L, 100, 200, width)
        qs = part.queues()
        if exp == "left":
            assert qid[0] == 0 and made == 0, L
        elif exp == "right":
            assert qid[0] == 1 and made == 0, L
        else:
            assert made == 1, L
            assert (qs[1]["min_len"], qs[1]["max_len"]) == exp, L
            assert qs[1]["min_len"] <= L < qs[1]["max_len"]
            assert qs[1]["mean"] == L                                  # R21


def test_bubble_edges_and_sequence(orc):
    """Below the first / above the last queue (R20); later gap requests see the
    bubbles created before them (R22, pool-index order); indices renumbered."""
    part = orc.make_partition([(100, 200), (400, 500)])
    s, qid, bad, made, _ = orc.route([10, 12, 300, 305, 900, 0, 150], part, 40)
    qs = part.queues()
    assert [(q["min_len"], q["max_len"]) for q in qs] == [(1, 30), (100, 200), (280, 320), (400, 500), (880, 920)]
    assert [q["index"] for q in qs] == [1, 2, 3, 4, 5]
    ids = {(q["min_len"]): q["id"] for q in qs}
    assert list(qid) == [ids[1], ids[1], ids[280], ids[280], ids[880], -1, ids[100]]
    assert bad == 1 and made == 3


def test_bubble_capacity(orc):
    part = orc.make_partition([(1000 + i, 1001 + i) for i in range(200)])
    lens = [int(1400 * 1.25 ** j) for j in range(62)]     # each > 1.1x the previous bubble
    s, qid, bad, made, dropped = orc.route(lens, part, 2)
    assert part.n == 256 and made == 56 and dropped == 6 and bad == 0 and s == orc.CAPACITY
    assert (qid[56:] == -1).all() and (qid[:56] >= 200).all()


# ------------------------------------------------------------ scoring (A10) ---
@pytest.mark.parametrize("ex", GOLD["score"], ids=lambda e: e["cite"][:20])
def test_score_golden(orc, ex):
    # W and C realised through now/arrival and a cost field
    sp = orc.select_params(now=float(ex["W"]))
    phi = orc.score_one(ex["b"], 0.0, ex["index"], ex["w"], sp, cost=ex["C"])
    assert phi == pytest.approx(ex["expected"], rel=1e-15)


@pytest.mark.parametrize("ex", GOLD["prefill_cost"], ids=lambda e: e["cite"])
def test_prefill_cost_golden(orc, ex):
    """C_prefill via the cost=NULL path: weights (0,1,0), index b+1, W=1 -> Φ = 1/C."""
    c = ex["c"]
    sp = orc.select_params(now=1.0, c0=c[0], c1=c[1], c2=c[2])
    phi = orc.score_one(ex["b"], 0.0, ex["b"] + 1, [0, 1, 0], sp)
    assert 1.0 / phi == pytest.approx(ex["expected"], rel=2e-7)       # fp32-stored coefficients


def test_score_exclusions(orc):
    sp = orc.select_params(now=10.0)
    assert orc.score_one(5, 11.0, 1, [1, 1, 1], sp, cost=1.0) is None       # W < 0
    assert orc.score_one(5, 1.0, 1, [1, 1, 1], sp, cost=0.0) is None        # C <= 0
    assert orc.score_one(5, float("nan"), 1, [1, 1, 1], sp, cost=1.0) is None
    assert orc.score_one(5, 10.0, 1, [1, 1, 1], sp, cost=1.0) is not None   # W = 0 ok


def test_score_vs_exact_rational(orc):
    rng = np.random.default_rng(3)
    for _ in range(500):
        b = int(rng.integers(1, 40000)); idx = int(rng.integers(1, 33))
        w = np.float32(rng.random(3) * 4)
        arr = np.float32(rng.random() * 600); cost = np.float32(rng.random() * 5 + 1e-3)
        sp = orc.select_params(now=600.0)
        got = orc.score_one(b, float(arr), idx, w, sp, cost=float(cost))
        W = Fr(float(np.float32(600.0))) - Fr(float(arr))
        ref = brute.score_exact(idx, b, W, Fr(float(cost)), float(w[0]), float(w[1]), float(w[2]))
        assert abs(Fr(got) - ref) <= abs(ref) * Fr(1, 10 ** 13)


@settings(max_examples=500, deadline=None)
@given(st.integers(1, 32768), st.integers(1, 64), st.floats(0.0, 5.0), st.floats(1e-3, 5.0),
       st.floats(0.0, 5.0), st.floats(0.0, 500.0), st.floats(0.01, 100.0), st.floats(1e-3, 10.0))
def test_starvation_freedom_monotone_unbounded(orc, b, idx, wb, wu, wf, arr, delta, cost):
    """Acceptance #4: with w_urg > 0 the score strictly
    increases with now, and the closed-form inversion W* reaches any target."""
    w = np.float32([wb, wu, wf])
    now1 = np.float32(arr + 1.0)
    now2 = np.float32(now1 + delta)
    p1 = orc.score_one(b, arr, idx, w, orc.select_params(now=float(now1)), cost=cost)
    p2 = orc.score_one(b, arr, idx, w, orc.select_params(now=float(now2)), cost=cost)
    assert p2 > p1
    target = p1 * 1000.0 + 1.0
    qf = idx / (b + 1.0)
    c32 = float(np.float32(cost))
    Wstar = (target / qf - float(w[0]) - float(w[2]) * math.log(b + 1.0)) * c32 / float(w[1])
    p3 = orc.score_one(b, 0.0, idx, w, orc.select_params(now=float(np.float32(Wstar * 1.001 + 1))), cost=cost)
    assert p3 >= target


def test_score_scale_covariance(orc):
    """weights × c multiply every score by c."""
    rng = np.random.default_rng(9)
    for _ in range(200):
        b = int(rng.integers(1, 5000)); w = rng.random(3).astype(np.float32)
        sp = orc.select_params(now=100.0)
        p = orc.score_one(b, 3.0, 4, w, sp, cost=0.7)
        q = orc.score_one(b, 3.0, 4, (w * np.float32(4.0)).astype(np.float32), sp, cost=0.7)
        assert q == pytest.approx(4.0 * p, rel=1e-15)


# ---------------------------------------------------------- selection (A11) ---
def _small_pool(rng, n):
    lens = rng.integers(1, 60, size=n).astype(np.int32)
    arr = np.float32(rng.integers(0, 8, size=n) * 0.5)          # many equal arrivals -> index ties
    cost = (rng.integers(1, 4, size=n) * 0.25).astype(np.float32)
    return lens, arr, cost


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("seed", range(25))
def test_select_vs_subset_enumeration(orc, mode, seed):
    """North_star: brute-force optimal selection agrees on pools of <= 20 requests."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 19))
    lens, arr, cost = _small_pool(rng, n)
    part = orc.make_partition([(1, 20), (20, 40), (40, 60)])
    K = int(rng.integers(1, 7))
    sp = orc.select_params(k=K, mode=mode, now=5.0)
    theta = orc.meta(a_b=0.01, b_b=0.2, a_u=-0.01, b_u=1.0, a_f=0.02, b_f=0.1)
    res = orc.tick(lens, arr, cost, part, theta, sp, global_base=1000)
    qid = res["qid"]
    for p in range(3):
        members = [r for r in range(n) if qid[r] == p]
        w = orc.weights(theta, part.q[p].mean)
        phi = {r: orc.score_one(int(lens[r]), float(arr[r]), p + 1, w, sp, cost=float(cost[r])) for r in members}
        members = [r for r in members if phi[r] is not None]
        assert res["count"][p] == len(members)
        if not members:
            assert res["topk_id"][p].tolist() == [-1] * K and res["head_id"][p] == -1
            continue
        keys = [(phi[r], -r) if mode == 0 else (-float(arr[r]), -r) for r in members]
        best = brute.topk_brute(keys, K)
        got = [int(i) - 1000 for i in res["topk_id"][p] if i >= 0]
        assert set(got) == {members[i] for i in best}
        # ordering: best first
        order = sorted(members, key=(lambda r: (-phi[r], r)) if mode == 0 else (lambda r: (float(arr[r]), r)))
        assert got == order[:K]
        head = min(members, key=lambda r: (float(arr[r]), r))
        assert res["head_id"][p] == head + 1000
        assert res["head_score"][p] == phi[head]
        assert res["max_score"][p] == max(phi.values() if not None else [])
    ne = [p for p in range(3) if res["count"][p] > 0]
    if ne:
        exp = max(ne, key=lambda p: (res["head_score"][p], -p))
        assert res["primary"] == exp
    else:
        assert res["primary"] == -1


def test_select_sjf_and_fcfs_degeneracies(orc):
    """One queue, weights (1,0,0): SCORE order is SJF (shortest first, ties by
    index).  FIFO mode with one queue is FCFS."""
    rng = np.random.default_rng(1)
    n = 300
    lens = rng.integers(1, 500, size=n).astype(np.int32)
    arr = np.float32(rng.random(n) * 10)
    part = orc.make_partition([(1, 1000)])
    theta = orc.meta(a_b=0, b_b=1, a_u=0, b_u=0, a_f=0, b_f=0)
    r = orc.tick(lens, arr, None, part, theta, orc.select_params(k=300, mode=0, now=20.0))
    np.testing.assert_array_equal(r["topk_id"][0], np.lexsort((np.arange(n), lens)))
    r = orc.tick(lens, arr, None, part, theta, orc.select_params(k=300, mode=1, now=20.0))
    np.testing.assert_array_equal(r["topk_id"][0], np.lexsort((np.arange(n), arr)))


def test_tick_domain_and_invalid(orc):
    part = orc.make_partition([(1, 10), (10, 100)])
    lens = np.array([5, 0, 50, 7], np.int32)
    arr = np.float32([1.0, 1.0, 99.0, 2.0])
    r = orc.tick(lens, arr, None, part, orc.meta(), orc.select_params(k=2, now=10.0))
    assert r["status"] == orc.DOMAIN and r["n_invalid"] == 1 and r["n_excluded"] == 1
    assert r["qid"].tolist() == [0, -1, 1, 0]
    assert r["count"].tolist() == [2, 0]
    assert r["primary"] == 0


def test_alpha_monotonicity_is_per_node_only(orc):
    """S:183 claims raising α never increases the number of splits.  With the
    per-sub-cluster mean(G) of S:192 (R12) that holds at one node but not for the
    whole recursion; the exact-rational literal Eq. 2 agrees with the oracle on a
    counterexample (recorded in DESIGN.md §3)."""
    xs = [157, 293, 19, 67, 139, 150, 290, 119, 125]
    assert len(orc.refine(xs, 1.5)) == len(brute.refine_brute(xs, 1.5)) == 3
    assert len(orc.refine(xs, 2.0)) == len(brute.refine_brute(xs, 2.0)) == 4
    rng = np.random.default_rng(0)
    for _ in range(500):     # one node: the qualifying-gap set shrinks as alpha grows
        v = np.sort(rng.integers(1, 300, size=int(rng.integers(2, 40))))
        g = np.diff(v); n = len(v); span = int(v[-1] - v[0])
        prev = None
        for a in (1.25, 1.5, 2.0, 3.0, 5.0):
            cur = {int(j) for j in np.nonzero(g * (n - 1) > a * span)[0]}
            assert prev is None or cur <= prev
            prev = cur


# ------------------------------------------------------------ Θ sweep (A12) ---
_SPECIAL_THETAS = [
    dict(a_b=0, b_b=1, a_u=0, b_u=0, a_f=0, b_f=0),        # SJF within a queue
    dict(a_b=0, b_b=0, a_u=0, b_u=1, a_f=0, b_f=0),        # urgency only
    dict(a_b=0, b_b=0, a_u=0, b_u=0, a_f=0, b_f=1),        # fairness only
    dict(a_b=-1, b_b=0, a_u=-1, b_u=0, a_f=-1, b_f=0),     # all weights clamp to 0: ids decide
    dict(a_b=0.01, b_b=0.2, a_u=-0.01, b_u=1.0, a_f=0.02, b_f=0.1),
]


@pytest.mark.parametrize("seed", range(12))
def test_sweep_vs_subset_enumeration(orc, seed):
    """O11: every Θ of the sweep selects the brute-force optimal top-K subset
    (pools of <= 20 requests, exact rational Eq. 4 up to the log term)."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 19))
    lens, arr, cost = _small_pool(rng, n)
    part = orc.make_partition([(1, 20), (20, 40), (40, 60)])
    s, qid, *_ = orc.route(lens, orc.copy_partition(part), 64)
    K = int(rng.integers(1, 6))
    sp = orc.select_params(k=K, mode=0, now=5.0)
    thetas = _SPECIAL_THETAS + [dict(zip(("a_b", "b_b", "a_u", "b_u", "a_f", "b_f"),
                                         rng.uniform([-0.05, 0, -0.05, 0, -0.05, 0], [0.05, 2, 0.05, 2, 0.05, 2])))
                                for _ in range(3)]
    st_, res = orc.sweep(lens, arr, cost, qid, part, thetas, sp, global_base=7)
    assert len(res) == len(thetas)
    for th, r in zip(thetas, res):
        ne = []
        for p in range(3):
            w = orc.weights(orc.meta(**th), part.q[p].mean)
            members = [i for i in range(n) if qid[i] == part.q[p].id]
            exact = {i: brute.score_exact(p + 1, int(lens[i]), F32(5.0) - F32(arr[i]), F32(cost[i]),
                                          F32(w[0]), F32(w[1]), F32(w[2])) for i in members}
            assert r["count"][p] == len(members)
            if not members:
                assert r["topk_id"][p].tolist() == [-1] * K
                continue
            ne.append(p)
            best = brute.topk_brute([(exact[i], -i) for i in members], K)
            got = [int(g) - 7 for g in r["topk_id"][p] if g >= 0]
            assert set(got) == {members[j] for j in best}, th
            assert got == sorted(got, key=lambda i: (-exact[i], i))
            for g, sc in zip(got, r["topk_score"][p]):
                assert sc == pytest.approx(float(exact[g]), rel=1e-12, abs=1e-300)
        if ne:
            assert r["primary"] == max(ne, key=lambda p: (r["head_score"][p], -p))


def F32(x):
    return Fr(float(np.float32(x)))


def test_sweep_special_cases_reduce_to_sorts(orc):
    """Θ = (1,0,0) is SJF: per queue, ascending length then id.  All-zero weights:
    every Φ = 0, so ascending id.  Doubling Θ doubles every weight exactly
    (fp64 a·mean + b and the fp32 rounding commute with ×2) so ids are
    unchanged and every score doubles exactly (Eq. 4 is linear in w)."""
    rng = np.random.default_rng(3)
    n = 2000
    lens = rng.integers(1, 600, size=n).astype(np.int32)
    arr = np.float32(rng.random(n) * 50)
    part = orc.make_partition([(1, 100), (100, 300), (300, 1000)])
    s, qid, *_ = orc.route(lens, orc.copy_partition(part), 64)
    th = [_SPECIAL_THETAS[0], _SPECIAL_THETAS[3], _SPECIAL_THETAS[4],
          {k: 2 * v for k, v in _SPECIAL_THETAS[4].items()}]
    st_, res = orc.sweep(lens, arr, None, qid, part, th, orc.select_params(k=50, mode=0, now=60.0))
    for p in range(3):
        idx = np.nonzero(qid == part.q[p].id)[0]
        sjf = idx[np.lexsort((idx, lens[idx]))][:50]
        np.testing.assert_array_equal(res[0]["topk_id"][p], sjf)
        np.testing.assert_array_equal(res[1]["topk_id"][p], idx[:50])
        assert (res[1]["topk_score"][p] == 0).all()
        np.testing.assert_array_equal(res[3]["topk_id"][p], res[2]["topk_id"][p])
        np.testing.assert_array_equal(res[3]["topk_score"][p], 2 * res[2]["topk_score"][p])
        assert res[3]["head_score"][p] == 2 * res[2]["head_score"][p]
    assert res[1]["primary"] == 0                       # all head scores 0 -> lowest position (R24)


# ------------------------------------------------ O12: Alg. 1 Batch Builder ---
def _bpool(orc, specs, now=100.0):
    """specs: [(len, arrival)], routed onto queues [1,100) [100,200) [200,300)."""
    part = orc.make_partition([(1, 100), (100, 200), (200, 300)])
    lens = np.array([b for b, _ in specs], np.int32)
    arr = np.array([a for _, a in specs], np.float32)
    s, qid, *_ = orc.route(lens, orc.copy_partition(part), 64)
    return part, lens, arr, qid, orc.select_params(k=8, mode=1, now=now)


def test_batch_spec_examples(orc):
    """all empty -> empty batch; one queue, 3 fitting requests -> those 3
    in FIFO order; primary's single request uses half the token budget and the
    neighbour has 2 fitting requests -> 3, neighbour's appended."""
    part, lens, arr, qid, sp = _bpool(orc, [])
    ids, tok = orc.batch(lens, arr, None, qid, part, sp, -1, 8, 1000)
    assert list(ids) == [] and tok == 0
    p2, e, removed = orc.prune_empty(part, [0, 0, 0], [0, 0, 0], 5)
    assert list(e) == [1, 1, 1] and removed == 0
    part, lens, arr, qid, sp = _bpool(orc, [(50, 3.0), (60, 1.0), (70, 2.0)])
    ids, tok = orc.batch(lens, arr, None, qid, part, sp, 0, 8, 1000)
    assert list(ids) == [1, 2, 0] and tok == 180          # FIFO by arrival
    part, lens, arr, qid, sp = _bpool(orc, [(150, 1.0), (40, 2.0), (30, 3.0)])
    ids, tok = orc.batch(lens, arr, None, qid, part, sp, 1, 8, 300)   # 150 = half of 300
    assert list(ids) == [0, 1, 2] and tok == 220


def test_batch_first_request_always_admitted_and_fifo_stop(orc):
    """the batch's first request is admitted even above max_tokens; a queue
    is pulled while the budget admits (R28: stop at the first that does not fit,
    no skipping ahead in its FIFO)."""
    part, lens, arr, qid, sp = _bpool(orc, [(250, 1.0), (20, 2.0)])
    ids, tok = orc.batch(lens, arr, None, qid, part, sp, 2, 8, 100)
    assert list(ids) == [0] and tok == 250                # oversized first request alone
    part, lens, arr, qid, sp = _bpool(orc, [(10, 1.0), (90, 2.0), (5, 3.0), (120, 4.0)])
    ids, tok = orc.batch(lens, arr, None, qid, part, sp, 0, 8, 50)
    # primary [10, 90, 5]: 10 fits, 90 does not -> stop (5 is not taken); backfill
    # queue 1 (distance 1, no lower neighbour): 120 does not fit
    assert list(ids) == [0] and tok == 10


def test_batch_backfill_nearest_lower_first_and_caps(orc):
    """R29: backfill visits index distance 1, 2, ..., lower neighbour
    first, FIFO within each queue; max_requests caps the batch."""
    part = orc.make_partition([(1, 10), (10, 20), (20, 30), (30, 40), (40, 50)])
    specs = [(45, 1.0), (35, 2.0), (25, 3.0), (15, 4.0), (5, 5.0), (26, 6.0), (14, 7.0), (44, 8.0)]
    lens = np.array([b for b, _ in specs], np.int32)
    arr = np.array([a for _, a in specs], np.float32)
    s, qid, *_ = orc.route(lens, orc.copy_partition(part), 64)
    sp = orc.select_params(k=8, mode=1, now=100.0)
    ids, tok = orc.batch(lens, arr, None, qid, part, sp, 2, 16, 10_000)
    # primary 2: [25(r2), 26(r5)]; d=1: queue 1 [15(r3), 14(r6)], queue 3 [35(r1)];
    # d=2: queue 0 [5(r4)], queue 4 [45(r0), 44(r7)]
    assert list(ids) == [2, 5, 3, 6, 1, 4, 0, 7]
    assert tok == int(lens.sum())
    ids, _ = orc.batch(lens, arr, None, qid, part, sp, 2, 3, 10_000)
    assert list(ids) == [2, 5, 3]


def test_batch_invariants_random(orc):
    """Every queue contributes a FIFO prefix of its members; count <= max_requests;
    tokens <= max_tokens unless the batch is one request; the primary's prefix is
    maximal; members are exactly the scored requests (W >= 0)."""
    import workload
    rng = np.random.default_rng(12)
    part = orc.make_partition(workload.quantile_bounds(workload.heavy(20_000, 3), 8))
    for trial in range(30):
        n = int(rng.integers(1, 400))
        lens = workload.heavy(n, 100 + trial)
        arr = (rng.random(n) * 120).astype(np.float32)         # some arrive after now: excluded
        s, qid, *_ = orc.route(lens, orc.copy_partition(part), 64)
        sp = orc.select_params(k=8, mode=1, now=100.0)
        mr = int(rng.integers(1, 40)); mt = int(rng.integers(100, 20_000))
        prim = int(rng.integers(0, part.n))
        ids, tok = orc.batch(lens, arr, None, qid, part, sp, prim, mr, mt)
        assert len(ids) <= mr and len(set(ids)) == len(ids)
        assert tok == int(lens[ids].sum()) if len(ids) else tok == 0
        assert tok <= mt or len(ids) == 1
        pos = {part.q[i].id: i for i in range(part.n)}
        for p in range(part.n):
            mem = [r for r in range(n) if qid[r] >= 0 and pos[qid[r]] == p and arr[r] <= 100.0]
            mem.sort(key=lambda r: (float(arr[r]), r))
            got = [int(r) for r in ids if pos[qid[r]] == p]
            assert got == mem[:len(got)], (trial, p)
            if p == prim and len(got) < len(mem) and len(ids) < mr:
                nxt = mem[len(got)]
                prim_tok = int(lens[[r for r in ids if pos[qid[r]] == p]].sum())
                assert prim_tok + int(lens[nxt]) > mt   # the next primary member did not fit


def test_prune_empty_threshold_strict_and_renumbers(orc):
    """Alg. 1 lines 8-12: empty queues count up, a queue with members resets its
    counter (consecutive empty steps, R30); removal when the counter exceeds
    the threshold (strict, R25); indices renumbered."""
    part = orc.make_partition([(1, 10), (10, 20), (20, 30), (30, 40)])
    e = [5, 0, 4, 5]
    p2, e2, removed = orc.prune_empty(part, e, [0, 0, 0, 7], 5)
    # queue 0: 5 -> 6 > 5 removed; queue 1: 0 -> 1; queue 2: 4 -> 5 kept; queue 3 non-empty: reset to 0
    assert removed == 1
    assert [(q["min_len"], q["index"]) for q in p2.queues()] == [(10, 1), (20, 2), (30, 3)]
    assert list(e2) == [1, 5, 0]


# ------------------------------------------------- O13: online adjust (R31) ---
def _counted(orc, bounds, counts):
    p = orc.make_partition(bounds)
    for i, c in enumerate(counts):
        p.q[i].count = c
    return p


def test_online_adjust_hand_example(orc):
    """Window entirely inside queue [10,20): only that queue's two boundaries move
    (S:178), each clamped to floor(0.25 * adjacent width) = 2: local targets 13
    (k = ceil(4*10/20) = 2 -> v_1 + 1) for both."""
    p = _counted(orc, [(1, 10), (10, 20), (20, 30)], [10, 10, 10])
    p2, moved = orc.online_adjust([12, 12, 12, 12], p, 0.25)
    assert moved == 2
    assert [(q["min_len"], q["max_len"]) for q in p2.queues()] == [(1, 12), (12, 18), (18, 30)]
    p3, moved = orc.online_adjust([15, 16, 17, 18, 25], _counted(orc, [(1, 10), (10, 20), (20, 30)], [0, 10, 10]), 0.25)
    # boundary 10: c_a = 0 -> k = 0 -> T = L = 1, clamped to 10 - floor(0.25*9) = 8;
    # boundary 20: members 15..18, 25 -> k = ceil(5*10/20) = 3 -> T = 18, d = -2 (limit 2)
    assert [(q["min_len"], q["max_len"]) for q in p3.queues()] == [(1, 8), (8, 18), (18, 30)]
    assert moved == 2


def test_online_adjust_identity_cases(orc):
    p = _counted(orc, [(1, 10), (10, 20), (20, 30)], [10, 10, 10])
    for w, s in (([], 0.25), ([5, 15, 25] * 10, 0.0), ([0, -3], 0.25)):
        p2, moved = orc.online_adjust(np.array(w, np.int32), p, s)
        assert moved == 0 and [(q["min_len"], q["max_len"]) for q in p2.queues()] == [(1, 10), (10, 20), (20, 30)]


def _adjust_brute(bounds, counts, window, s):
    """The definition searched over every x (no order-statistic closed form)."""
    new = [b[0] for b in bounds] + [bounds[-1][1]]
    out = list(new)
    for i in range(1, len(bounds)):
        L, B, U = bounds[i - 1][0], bounds[i][0], bounds[i][1]
        if bounds[i - 1][1] != B:
            continue
        ca, cb = counts[i - 1], counts[i]
        loc = [w for w in window if w >= 1 and L <= w < U]
        m = len(loc)
        if m == 0 or ca + cb == 0:
            continue
        T = next(x for x in range(L, U + 1) if sum(v < x for v in loc) * (ca + cb) >= m * ca)
        d = max(-math.floor(s * (B - L)), min(math.floor(s * (U - B)), T - B))
        out[i] = B + d
    return out


@settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.lists(st.integers(1, 12), min_size=1, max_size=6), st.lists(st.integers(0, 20), min_size=6, max_size=6),
       st.lists(st.integers(-2, 80), max_size=40), st.sampled_from([0.0, 0.1, 0.25, 0.4, 0.49]))
def test_online_adjust_matches_definition_and_invariants(orc, widths, counts, window, s):
    b, bounds = 1, []
    for w in widths:
        bounds.append((b, b + w)); b += w
    counts = counts[: len(bounds)]
    p = _counted(orc, bounds, counts)
    p2, moved = orc.online_adjust(np.array(window, np.int32), p, s)
    q2 = p2.queues()
    edges = [q2[0]["min_len"]] + [q["max_len"] for q in q2]
    assert edges == _adjust_brute(bounds, counts, window, s)
    assert all(q["max_len"] > q["min_len"] for q in q2)                        # width >= 1, order kept
    assert all(q2[i]["max_len"] == q2[i + 1]["min_len"] for i in range(len(q2) - 1))
    assert moved == sum(e != o for e, o in zip(edges, [bb[0] for bb in bounds] + [bounds[-1][1]]))


def test_online_adjust_same_distribution_is_near_identity(orc):
    """a window drawn like the history moves each boundary by little; under
    quantile matching an interior boundary with mass on both sides moves by at
    most a few lengths (here the 32-quantile partition of heavy(200k))."""
    import workload
    hist = workload.heavy(200_000, 3)
    bounds = workload.quantile_bounds(hist, 16)
    counts = [int(((hist >= lo) & (hist < hi)).sum()) for lo, hi in bounds]
    p = _counted(orc, bounds, counts)
    p2, _ = orc.online_adjust(workload.heavy(200_000, 4), p, 0.25)
    for (lo, hi), q in zip(bounds, p2.queues()):
        w = hi - lo
        assert abs(q["min_len"] - lo) <= max(2, 0.05 * w)


# ---------------------------------- Eq. 2 over the set of distinct lengths ---
def test_gap_rule_set_reading_example(orc):
    """SURVEY ambiguity 10: G over the multiset D (R10, default) vs over the set of
    distinct lengths (gap_rule=1).  [1 x6, 2, 10], alpha = 2: the multiset reading
    splits twice (mean(G) = 9/7, then 1/6), the set reading {1, 2, 10} not at all
    (mean(G) = 4.5, gap 8 < 9)."""
    xs = [1] * 6 + [2, 10]
    s0, _, st0 = orc.partition(xs, coarse_k=1, max_queues=256)
    s1, _, st1 = orc.partition(xs, coarse_k=1, max_queues=256, gap_rule=1)
    assert st0.segments == len(brute.refine_brute(xs, 2.0)) == 3
    assert st1.segments == len(brute.refine_brute(sorted(set(xs)), 2.0)) == 1


@settings(max_examples=80, deadline=None)
@given(st.lists(st.integers(1, 60), min_size=1, max_size=40), st.sampled_from([1.5, 2.0, 3.0]))
def test_gap_rule_set_matches_brute_on_distinct_values(orc, xs, alpha):
    s, _, st_ = orc.partition(xs, coarse_k=1, max_queues=256, alpha=alpha, gap_rule=1)
    assert st_.segments == len(brute.refine_brute(sorted(set(xs)), alpha))


def _midpoint_bounds(clusters):
    """A5 finalisation (R15) of Stage-2 clusters given as sorted value lists:
    B_0 = lo_1, B_i = floor((hi_i + lo_{i+1}) / 2) + 1, B_m = hi_m + 1."""
    lo = [c[0] for c in clusters]
    hi = [c[-1] for c in clusters]
    B = [lo[0]] + [(hi[i] + lo[i + 1]) // 2 + 1 for i in range(len(clusters) - 1)] + [hi[-1] + 1]
    return list(zip(B[:-1], B[1:]))


@settings(max_examples=120, deadline=None)
@given(st.lists(st.integers(1, 80), min_size=1, max_size=40), st.sampled_from([1.5, 2.0, 3.0]),
       st.sampled_from([0, 1]))
def test_refine_cut_positions_match_brute(orc, xs, alpha, gap_rule):
    """Eq. 2 cut POSITIONS, both gap readings (R10 multiset / SURVEY ambiguity 10
    set): with one coarse cluster and no pruning (<= 40 items, max_queues = 256) the oracle's
    queue bounds are the midpoint finalisation of brute.refine_brute's clusters (exact
    rational Eq. 2 over the explicit gap list — the multiset, or the set of distinct
    lengths), and every queue holds exactly its cluster's members."""
    s, part, st_ = orc.partition(xs, coarse_k=1, max_queues=256, alpha=alpha, gap_rule=gap_rule)
    assert s == orc.OK
    base = sorted(xs) if gap_rule == 0 else sorted(set(xs))
    clusters = brute.refine_brute(base, alpha)
    qs = part.queues()
    assert [(q["min_len"], q["max_len"]) for q in qs] == _midpoint_bounds(clusters)
    v = np.asarray(xs)
    for q, c in zip(qs, clusters):
        assert q["count"] == int(((v >= c[0]) & (v <= c[-1])).sum())


def test_refine_set_reading_cut_positions_example(orc):
    """[1 x6, 2, 10, 11, 30]: multiset mean(G) = 29/9 splits at 10-2=8 and 30-11=19
    (> 2 * 29/9 = 6.44); the set {1, 2, 10, 11, 30} has mean(G) = 29/4 and only 19 > 14.5
    qualifies.  Bounds after the midpoint rule: multiset [1,7) [7,21) [21,31) ... checked
    against the brute force and by hand."""
    xs = [1] * 6 + [2, 10, 11, 30]
    _, p0, _ = orc.partition(xs, coarse_k=1, max_queues=256)
    _, p1, _ = orc.partition(xs, coarse_k=1, max_queues=256, gap_rule=1)
    b0 = [(q["min_len"], q["max_len"]) for q in p0.queues()]
    b1 = [(q["min_len"], q["max_len"]) for q in p1.queues()]
    # multiset: gaps [0,0,0,0,0,1,8,1,19], mean 29/9, threshold 58/9 = 6.44 -> cuts after 2 and 11;
    # {1x6, 2} then mean(G) = 1/6 -> split 1 | 2; {10, 11}: mean 1, gap 1 not > 2 -> stays
    assert b0 == [(1, 2), (2, 7), (7, 21), (21, 31)]
    # set: gaps [1, 8, 1, 19], mean 29/4, threshold 14.5 -> cut after 11 only; {1,2,10,11}: mean 10/3,
    # threshold 20/3 -> 8 qualifies -> {1,2} | {10,11}; {1,2}: one gap = mean -> no split
    assert b1 == [(1, 7), (7, 21), (21, 31)]
