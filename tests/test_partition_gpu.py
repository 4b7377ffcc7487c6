"""GPU Refine-and-Prune (ewsjf_partition) vs the CPU oracle: bit-exact boundaries,
integer profiles, fp64 means/densities and every pipeline statistic."""
import numpy as np
import pytest
import torch

import workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import paper_2601_21758_b200 as E
    return E


@pytest.fixture(scope="module")
def ctx(E):
    return E.Context(0, max_pool=1024, max_history=100_000_000, max_k=8)


def _both(E, orc, ctx, hist, **kw):
    h = np.ascontiguousarray(hist, dtype=np.int32)
    gpart, gst, gs = E.partition(ctx, torch.from_numpy(h).cuda(), E.partition_params(**kw))
    os_, opart, ost = orc.partition(h, **kw)
    return gpart, gst, gs, opart, ost, os_


def _check(gpart, gst, gs, opart, ost, os_):
    assert gs == os_, (gs, os_)
    gq, oq = gpart.queues(), opart.queues()
    keys = ("id", "index", "min_len", "max_len", "count", "sum", "sumsq", "mean", "density", "sse", "is_bubble")
    assert len(gq) == len(oq)
    for a, b in zip(gq, oq):
        for k in keys:
            assert a[k] == b[k], (k, a, b)          # bit-exact, fp64 included
    for k in ("n_valid", "n_invalid", "distinct", "k_used", "t1", "t2", "segments", "depth", "merges"):
        assert gst[k] == getattr(ost, k), (k, gst[k], getattr(ost, k))


@pytest.mark.parametrize("kind,n,seed", [("bimodal", 10_000, 101), ("heavy", 10_000, 7), ("bimodal", 200_000, 3),
                                         ("heavy", 300_000, 4)])
@pytest.mark.parametrize("rule", [0, 1])
def test_partition_matches_oracle(E, orc, ctx, kind, n, seed, rule):
    _check(*_both(E, orc, ctx, workload.lengths(kind, n, seed), merge_rule=rule))


@pytest.mark.parametrize("seed", range(30))
def test_partition_random_small(E, orc, ctx, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    hi = int(rng.choice([5, 50, 500, 5000, 70000]))
    hist = rng.integers(1, hi, size=n)
    if seed % 5 == 0:
        hist[rng.integers(0, n, size=max(1, n // 20))] = 0        # invalid lengths
    kw = dict(alpha=float(rng.choice([1.5, 2.0, 3.0, 1.7])), min_width=int(rng.choice([1, 2, 10])),
              max_queues=int(rng.integers(1, 40)), epsilon=float(rng.choice([1e-6, 0.5, 2.0])),
              coarse_k=int(rng.integers(1, 4)), merge_rule=int(rng.integers(0, 2)),
              gap_rule=int(seed % 3 == 2))
    _check(*_both(E, orc, ctx, hist, **kw))


def test_partition_edge_cases(E, orc, ctx):
    for hist in ([777] * 50, [5, 6], [1], [3, 3, 9, 9, 9], [1, 2, 3, 4], list(range(1, 600))):
        _check(*_both(E, orc, ctx, np.array(hist)))
    g, st, s = E.partition(ctx, torch.zeros(10, dtype=torch.int32, device="cuda"))
    assert s == 3                                                  # EMPTY


def test_partition_full_c2(E, orc, ctx):
    """C2 history: 1M bimodal lengths (seed 201), default parameters."""
    _check(*_both(E, orc, ctx, workload.bimodal(1_000_000, 201)))


def test_partition_full_c3_history(E, orc, ctx):
    """The 1M heavy-tailed history bench.py partitions (seed 301)."""
    _check(*_both(E, orc, ctx, workload.heavy(1_000_000, 301)))


def test_partition_full_c4_bimodal(E, orc, ctx):
    """C4 at full size: Refine-and-Prune of a 100M bimodal history (seed 401)."""
    _check(*_both(E, orc, ctx, workload.bimodal(100_000_000, 401)))


def test_partition_full_c4_heavy(E, orc, ctx):
    """C4 at full size, the benched input: a 100M heavy-tailed history (seed 402,
    32,631 distinct lengths, 32,599 Stage-3 merges)."""
    _check(*_both(E, orc, ctx, workload.heavy(100_000_000, 402)))


@pytest.mark.parametrize("rule", [0, 1])
@pytest.mark.parametrize("top", [12_000, 18_000, 25_000, 40_000])
def test_partition_many_segments(E, orc, ctx, rule, top):
    """Every distinct length twice: each unit gap exceeds alpha * mean(G) ~ 1.0, so
    Stage 2 leaves `top` segments and Stage 3 merges them down to 32.  12k-18k
    segments run the all-shared-memory prune, 25k-40k the one with global
    leaves (C4's 100M heavy history has 32.6k)."""
    hist = np.repeat(np.arange(1, top + 1, dtype=np.int32), 2)
    g = _both(E, orc, ctx, hist, merge_rule=rule)
    assert g[1]["segments"] == top
    _check(*g)


def test_partition_many_segments_global_tree(E, orc, ctx):
    """56k segments: beyond both shared-memory variants -> global-memory tree."""
    hist = np.repeat(np.arange(1, 56_001, dtype=np.int32), 2)
    g = _both(E, orc, ctx, hist)
    assert g[1]["segments"] == 56_000
    _check(*g)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind,n,seed", [("heavy", 300_000, 11), ("bimodal", 100_000, 12)])
def test_partition_from_summed_shard_histograms(E, orc, ctx, world, kind, n, seed):
    """Sharded history: the per-shard histograms summed (what
    the NCCL all-reduce computes) give the partition of the whole history, bit for
    bit, equal to the oracle's."""
    h = workload.lengths(kind, n, seed).astype(np.int32)
    h[::997] = 0                                                  # a few invalid lengths
    dev = torch.from_numpy(h).cuda()
    tot = None
    inv, mx = 0, 0
    for r in range(world):
        a, b = workload.shard_range(n, r, world)
        hist, info = E.history_hist(ctx, dev[a:b].contiguous())
        tot = hist.clone() if tot is None else tot + hist
        inv += info["invalid"]; mx = max(mx, info["max_len"])
    gpart, gst, gs = E.partition_from_hist(ctx, tot, mx, inv)
    fpart, fst, fs = E.partition(ctx, dev)
    assert gs == fs
    assert [tuple(q.values()) for q in gpart.queues()] == [tuple(q.values()) for q in fpart.queues()]
    for k in ("n_valid", "n_invalid", "distinct", "segments", "merges"):
        assert gst[k] == fst[k], k
    os_, opart, ost = orc.partition(h)
    _check(gpart, gst, gs, opart, ost, os_)


def test_partition_from_hist_edge_cases(E, ctx):
    z = torch.zeros(E.HIST_BINS + 1, dtype=torch.int32, device="cuda")
    _, _, s = E.partition_from_hist(ctx, z, 0)
    assert s == 3                                                  # EMPTY
    _, _, s = E.partition_from_hist(ctx, z, 100)                   # max_len given, no mass
    assert s == 3


@pytest.mark.parametrize("kind,n,seed", [("heavy", 1_000_000, 301), ("bimodal", 200_000, 3)])
@pytest.mark.parametrize("rule", [0, 1])
def test_partition_set_gap_reading(E, orc, ctx, kind, n, seed, rule):
    """gap_rule = 1 (Eq. 2 over the set of distinct lengths, SURVEY ambiguity 10)."""
    _check(*_both(E, orc, ctx, workload.lengths(kind, n, seed), merge_rule=rule, gap_rule=1))


# ---- Table 3 "EWSJF (K-Means)": k-means-only partitions (oracle O14, R32)
def _check_kmeans(E, orc, ctx, hist, k):
    h = np.ascontiguousarray(hist, dtype=np.int32)
    gpart, gst, gs = E.partition(ctx, torch.from_numpy(h).cuda(), E.partition_params(kmeans_k=k))
    os_, opart, ost = orc.partition_kmeans(h, k)
    assert gs == os_, (gs, os_)
    gq, oq = gpart.queues(), opart.queues()
    assert len(gq) == len(oq) == ost.k_used == gst["k_used"]
    for a, b in zip(gq, oq):
        for key in ("id", "index", "min_len", "max_len", "count", "sum", "sumsq", "mean", "density", "sse"):
            assert a[key] == b[key], (key, a, b)    # bit-exact (the fp64 DP decisions included)


@pytest.mark.parametrize("k", [5, 10, 30])
@pytest.mark.parametrize("kind,n,seed", [("bimodal", 10_000, 101), ("heavy", 50_000, 9)])
def test_kmeans_only_partition_matches_oracle(E, orc, ctx, kind, n, seed, k):
    _check_kmeans(E, orc, ctx, workload.lengths(kind, n, seed), k)


@pytest.mark.parametrize("k", [5, 10, 30])
def test_kmeans_only_partition_c2_history(E, orc, ctx, k):
    """The C2 history (bimodal 1M, seed 201; ~12.5k distinct lengths)."""
    _check_kmeans(E, orc, ctx, workload.bimodal(1_000_000, 201), k)


@pytest.mark.parametrize("seed", range(12))
def test_kmeans_only_random_small(E, orc, ctx, seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 400))
    hist = rng.integers(1, int(rng.choice([4, 30, 300, 5000])), size=n)
    if seed % 4 == 0:
        hist[0] = 0                                  # one invalid length: DOMAIN on both sides
    _check_kmeans(E, orc, ctx, hist, int(rng.integers(1, 12)))


# ---- A1 long tail: history lengths >= 2^20 (prompts of a million tokens and more) ----
def _with_long_tail(n, n_long, seed, lo=1 << 20, hi=1 << 23):
    rng = np.random.default_rng(seed)
    h = workload.lengths("heavy", n, seed).astype(np.int64)
    idx = rng.choice(n, size=n_long, replace=False)
    # a few repeated values too (runs of equal over-long lengths)
    vals = rng.integers(lo, hi, size=n_long)
    vals[: n_long // 4] = vals[0]
    h[idx] = vals
    return h.astype(np.int32)


@pytest.mark.parametrize("n,n_long,seed", [(200_000, 1000, 11), (50_000, 32_768, 12), (3_000, 1, 13)])
def test_partition_long_prompt_tail(E, orc, ctx, n, n_long, seed):
    """Lengths >= 2^20 go through the overflow list (sorted in one CTA, RLE appended after
    the histogram's runs): same boundaries and statistics as the oracle's std::sort."""
    _check(*_both(E, orc, ctx, _with_long_tail(n, n_long, seed)))


def test_partition_only_long_prompts(E, orc, ctx):
    rng = np.random.default_rng(14)
    h = rng.integers(1 << 20, 1 << 30, size=5000).astype(np.int32)
    _check(*_both(E, orc, ctx, h))


def test_partition_long_tail_over_capacity_refused(E, ctx):
    h = _with_long_tail(100_000, 32_769, 15)
    with pytest.raises(E.EwsjfError) as ei:
        E.partition(ctx, torch.from_numpy(h).cuda())
    assert ei.value.status == 6          # EWSJF_ERR_UNSUPPORTED


def test_tick_routes_long_prompts(E, orc, ctx):
    """A partition with queues above 2^20 routes and scores long pending prompts like the oracle
    (lengths past the fused tick's LUT take its binary search)."""
    from tests.parity import compare_selection, gpu_result, to_gpu_partition
    hist = _with_long_tail(100_000, 2000, 16)
    s, opart, _ = orc.partition(hist)
    assert s == orc.OK
    pool = workload.pool("heavy", 200_000, 17)
    rng = np.random.default_rng(18)
    sel = rng.choice(200_000, size=3000, replace=False)
    pool["len"][sel] = rng.integers(1 << 20, 1 << 23, size=3000).astype(np.int32)
    tctx = E.Context(0, max_pool=200_000, max_history=0, max_k=64)
    qid = torch.empty(200_000, dtype=torch.int32, device="cuda")
    out = E.tick(tctx, *(torch.from_numpy(pool[k]).cuda() for k in ("len", "arrival", "cost")),
                 to_gpu_partition(E, opart), E.meta(**workload.THETA0), E.select_params(k=64, mode=0), qid_out=qid)
    ref = orc.tick(pool["len"], pool["arrival"], pool["cost"], opart, orc.meta(**workload.THETA0),
                   orc.select_params(k=64, mode=0))
    phi, _ = orc.score_all(pool["len"], pool["arrival"], pool["cost"], ref["qid"], ref["partition"],
                           orc.meta(**workload.THETA0), orc.select_params(k=64, mode=0))
    np.testing.assert_array_equal(qid.cpu().numpy(), ref["qid"])
    # every swap is still checked to lie within 1e-5 relative of the boundary score (north_star);
    # the count is not bounded here: at b ~ 2^22 the scores of adjacent lengths differ by
    # ~1/b = 2.4e-7 relative, about two fp32 ulps, so most of a long queue's top K are near-ties
    rep = compare_selection(gpu_result(out), ref, phi, pool["arrival"], 0, 64, near_tie_bound=None)
    print(f"long-prompt tick: {rep.near_ties} near-tie swaps over {rep.checked_queues} queues")
    tctx.close()
