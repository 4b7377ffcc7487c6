"""GPU parity of the fused tick / score_select / route against the CPU oracle.

Every case feeds identical seeded inputs (workload/) to the CUDA path (through
the C ABI) and to the oracle, and compares element by element (tests/parity.py).
"""
import numpy as np
import pytest
import torch

import workload
from tests.parity import compare_selection, gpu_result, to_gpu_partition, Report

pytestmark = pytest.mark.gpu

THETA0 = workload.THETA0


@pytest.fixture(scope="module")
def E():
    import paper_2601_21758_b200 as E
    return E


@pytest.fixture(scope="module")
def ctx(E):
    return E.Context(0, max_pool=1 << 22, max_history=1 << 21, max_k=256)


def _run_both(E, O, ctx, pool, opart, K, mode, bubble_width=64, base=0, now=600.0, cost_mode="field",
              shift=0):
    n = len(pool["len"])
    ln = torch.from_numpy(pool["len"]).cuda()
    ar = torch.from_numpy(pool["arrival"]).cuda()
    co = torch.from_numpy(pool["cost"]).cuda() if (pool["cost"] is not None and cost_mode == "field") else None
    if shift:   # misaligned views -> non-TMA path
        ln = torch.cat([torch.zeros(shift, dtype=ln.dtype, device="cuda"), ln])[shift:]
        ar = torch.cat([torch.zeros(shift, dtype=ar.dtype, device="cuda"), ar])[shift:]
        if co is not None:
            co = torch.cat([torch.zeros(shift, dtype=co.dtype, device="cuda"), co])[shift:]
    qid = torch.full((n + shift,), -7, dtype=torch.int32, device="cuda")[shift:]
    gpart = to_gpu_partition(E, opart)
    theta = E.meta(**THETA0)
    sp = E.select_params(k=K, mode=mode, now=now)
    out = E.tick(ctx, ln, ar, co, gpart, theta, sp, bubble_width=bubble_width, global_base=base, qid_out=qid)
    g = gpu_result(out)
    g["qid"] = qid.cpu().numpy()
    g["part"] = gpart
    ref = O.tick(pool["len"], pool["arrival"], pool["cost"] if co is not None else None, opart,
                 O.meta(**THETA0), O.select_params(k=K, mode=mode, now=now), bubble_width=bubble_width,
                 global_base=base)
    phi, valid = O.score_all(pool["len"], pool["arrival"], pool["cost"] if co is not None else None, ref["qid"],
                             ref["partition"], O.meta(**THETA0), O.select_params(k=K, mode=mode, now=now))
    return g, ref, phi


def _check(g, ref, phi, pool, mode, K, base=0):
    np.testing.assert_array_equal(g["qid"], ref["qid"], err_msg="qid (stable ids, exact)")
    assert g["n_bubbles"] == ref["n_bubbles"] and g["n_dropped"] == ref["n_dropped"]
    assert g["n_invalid"] == ref["n_invalid"] and g["n_excluded"] == ref["n_excluded"]
    oq = ref["partition"].queues()
    gq = g["part"].queues()
    assert [(q["min_len"], q["max_len"], q["id"]) for q in gq] == [(q["min_len"], q["max_len"], q["id"]) for q in oq]
    return compare_selection(g, ref, phi, pool["arrival"], mode, K, base)


@pytest.fixture(scope="module")
def c1_partition(orc):
    s, part, _ = orc.partition(workload.bimodal(10_000, 101))
    assert s == orc.OK
    return part


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("cost_mode", ["field", "params"])
def test_tick_c1(E, orc, ctx, c1_partition, mode, cost_mode):
    """C1: 1k bimodal pool, partition = Refine-and-Prune of the 10k bimodal history."""
    pool = workload.pool("bimodal", 1000, 102)
    g, ref, phi = _run_both(E, orc, ctx, pool, c1_partition, 64, mode, cost_mode=cost_mode)
    _check(g, ref, phi, pool, mode, 64)


@pytest.fixture(scope="module")
def heavy_parts(orc):
    hist = workload.heavy(200_000, 301)
    s, rp, _ = orc.partition(hist)
    assert s == orc.OK
    q = orc.make_partition(workload.quantile_bounds(hist, 32))
    return {"rp": rp, "quantile": q}


@pytest.mark.parametrize("which", ["rp", "quantile"])
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("K", [1, 64, 256])
def test_tick_tiles_ragged(E, orc, ctx, heavy_parts, which, mode, K):
    """Several TMA tiles per CTA plus a ragged tail (n = 148*2048*2 + 777)."""
    n = ctx.num_ctas * 2048 * 2 + 777
    pool = workload.pool("heavy", n, 302)
    g, ref, phi = _run_both(E, orc, ctx, pool, heavy_parts[which], K, mode)
    _check(g, ref, phi, pool, mode, K)


@pytest.mark.parametrize("mode", [0, 1])
def test_tick_shuffled_order(E, orc, ctx, heavy_parts, mode):
    """Arrival order uncorrelated with the index (worst case for the filters)."""
    pool = workload.pool("heavy", 300_001, 303, shuffled=True)
    g, ref, phi = _run_both(E, orc, ctx, pool, heavy_parts["quantile"], 64, mode, base=12345)
    _check(g, ref, phi, pool, mode, 64, base=12345)


@pytest.mark.parametrize("shift", [1, 3])
def test_tick_misaligned_views(E, orc, ctx, heavy_parts, shift):
    pool = workload.pool("heavy", 100_003, 304)
    g, ref, phi = _run_both(E, orc, ctx, pool, heavy_parts["rp"], 64, 0, shift=shift)
    _check(g, ref, phi, pool, 0, 64)


@pytest.mark.parametrize("mode", [0, 1])
def test_tick_gaps_and_bubbles(E, orc, ctx, mode):
    """A partition with holes: gap requests go through Alg. 2 in index order."""
    part = orc.make_partition([(32, 100), (180, 300), (1000, 2000), (5000, 6000)], means=[60, 240, 1500, 5500])
    rng = np.random.default_rng(7)
    n = 200_000         # ~130k gap requests through the epoch-parallel Alg. 2
    pool = {"len": rng.integers(1, 9000, size=n).astype(np.int32),
            "arrival": workload.arrivals(n, 7), "cost": workload.cost_estimates(np.ones(n, np.int32) * 100, 7)}
    g, ref, phi = _run_both(E, orc, ctx, pool, part, 16, mode, bubble_width=64)
    assert ref["n_bubbles"] > 10
    _check(g, ref, phi, pool, mode, 16)


def test_tick_all_pool_in_one_hole(E, ctx):
    """Every request falls in one hole (20k gap requests, far more than the old
    8192-entry list): the first creates the bubble [L - 32, L + 32), all the others
    land inside it (App. D Alg. 2 in index order) -- nothing is refused."""
    n = 20_000
    ln = torch.full((n,), 5000, dtype=torch.int32, device="cuda")
    ar = torch.zeros(n, dtype=torch.float32, device="cuda")
    qid = torch.empty(n, dtype=torch.int32, device="cuda")
    part = E.make_partition([(1, 10)])
    out = E.tick(ctx, ln, ar, None, part, E.meta(**THETA0), E.select_params(k=4), qid_out=qid)
    assert out.summary["status"] == 0 and out.summary["n_gap"] == n and out.summary["n_bubbles"] == 1
    assert (qid.cpu().numpy() == 1).all()
    assert [(q["min_len"], q["max_len"]) for q in part.queues()] == [(1, 10), (4968, 5032)]


def test_tick_bubble_cap(E, orc, ctx):
    """More gap lengths than queue slots: refusals at 256 queues (CAPACITY)."""
    part = orc.make_partition([(1000 + i, 1001 + i) for i in range(200)])
    lens = np.array([int(1400 * 1.25 ** j) for j in range(62)], np.int32)
    n = len(lens)
    pool = {"len": lens, "arrival": np.zeros(n, np.float32), "cost": np.ones(n, np.float32)}
    g, ref, phi = _run_both(E, orc, ctx, pool, part, 4, 0, bubble_width=2)
    assert g["n_dropped"] == 6 and g["status"] == 4
    _check(g, ref, phi, pool, 0, 4)


def test_tick_edge_values(E, orc, ctx, heavy_parts):
    """Invalid lengths, arrivals in the future, non-positive / NaN cost, -0.0 arrivals."""
    rng = np.random.default_rng(11)
    n = 20_000
    pool = workload.pool("heavy", n, 305)
    pool["len"][rng.integers(0, n, 300)] = 0
    pool["len"][rng.integers(0, n, 300)] = -5
    pool["arrival"][rng.integers(0, n, 300)] = 700.0
    pool["arrival"][rng.integers(0, n, 50)] = -0.0
    pool["cost"][rng.integers(0, n, 200)] = 0.0
    pool["cost"][rng.integers(0, n, 50)] = np.nan
    for mode in (0, 1):
        g, ref, phi = _run_both(E, orc, ctx, pool, heavy_parts["rp"], 32, mode)
        assert g["status"] == 2
        _check(g, ref, phi, pool, mode, 32)


@pytest.mark.parametrize("n", [0, 1, 3, 2047, 2048, 2049])
def test_tick_tiny_pools(E, orc, ctx, heavy_parts, n):
    pool = workload.pool("heavy", max(n, 1), 306)
    pool = {k: (v[:n] if v is not None else None) for k, v in pool.items()}
    for mode in (0, 1):
        g, ref, phi = _run_both(E, orc, ctx, pool, heavy_parts["rp"], 8, mode)
        _check(g, ref, phi, pool, mode, 8)


def test_tick_equal_scores_tiebreak(E, orc, ctx):
    """Identical requests: ties must go to the lowest id in both modes (R24, R26)."""
    n = 100_000
    pool = {"len": np.full(n, 500, np.int32), "arrival": np.full(n, 10.0, np.float32),
            "cost": np.full(n, 0.1, np.float32)}
    part = orc.make_partition([(1, 1000), (1000, 2000)])
    for mode in (0, 1):
        g, ref, phi = _run_both(E, orc, ctx, pool, part, 64, mode)
        np.testing.assert_array_equal(g["topk_id"][0], np.arange(64))
        _check(g, ref, phi, pool, mode, 64)


def test_route_matches_oracle(E, orc, ctx):
    part = orc.make_partition([(32, 100), (180, 300), (1000, 2000)])
    lens = np.random.default_rng(3).integers(-2, 4000, size=10_000).astype(np.int32)   # gaps < 8192
    gpart = to_gpu_partition(E, part)
    qid, summ = E.route(ctx, torch.from_numpy(lens).cuda(), gpart, 50)
    p2 = orc.copy_partition(part)
    s, oqid, bad, made, dropped = orc.route(lens, p2, 50)
    np.testing.assert_array_equal(qid.cpu().numpy(), oqid)
    assert summ["n_bubbles"] == made and summ["n_invalid"] == bad + dropped
    assert [(q["min_len"], q["max_len"], q["id"], q["index"]) for q in gpart.queues()] == \
           [(q["min_len"], q["max_len"], q["id"], q["index"]) for q in p2.queues()]


@pytest.mark.parametrize("mode", [0, 1])
def test_score_select_matches_oracle(E, orc, ctx, heavy_parts, mode):
    pool = workload.pool("bimodal", 250_000, 202)
    opart = heavy_parts["quantile"]
    s, oqid, *_ = orc.route(pool["len"], orc.copy_partition(opart), 64)
    w = np.stack([orc.weights(orc.meta(**THETA0), opart.q[i].mean) for i in range(opart.n)])
    gpart = to_gpu_partition(E, opart)
    import paper_2601_21758_b200._lib as L
    gw = (L.Weights * L.MAX_QUEUES)(*[L.Weights(*map(float, w[i])) for i in range(opart.n)])
    qd = torch.from_numpy(oqid).cuda()
    sp = E.select_params(k=32, mode=mode)
    out = E.score_select(ctx, torch.from_numpy(pool["len"]).cuda(), torch.from_numpy(pool["arrival"]).cuda(),
                         torch.from_numpy(pool["cost"]).cuda(), qd, gpart, gw, sp)
    ref = orc.score_select(pool["len"], pool["arrival"], pool["cost"], oqid, opart, w,
                           orc.select_params(k=32, mode=mode))
    phi, _ = orc.score_all(pool["len"], pool["arrival"], pool["cost"], oqid, opart, orc.meta(**THETA0),
                           orc.select_params(k=32, mode=mode))
    g = gpu_result(out)
    compare_selection(g, ref, phi, pool["arrival"], mode, 32)


def test_tick_host_equals_device(E, orc, ctx, heavy_parts):
    pool = workload.pool("heavy", 500_000, 307)
    gpart = to_gpu_partition(E, heavy_parts["rp"])
    theta, sp = E.meta(**THETA0), E.select_params(k=64)
    hl = torch.from_numpy(pool["len"]).pin_memory()
    ha = torch.from_numpy(pool["arrival"]).pin_memory()
    hc = torch.from_numpy(pool["cost"]).pin_memory()
    hq = torch.empty(len(hl), dtype=torch.int32).pin_memory()
    r = E.tick_host(ctx, hl, ha, hc, gpart, theta, sp, qid_out=hq)
    out = E.tick(ctx, hl.cuda(), ha.cuda(), hc.cuda(), to_gpu_partition(E, heavy_parts["rp"]), theta, sp)
    assert r["summary"] == out.summary
    nq = out.summary["n_queues"]
    for k in ("topk_id", "count", "head_id", "topk_score", "head_score", "max_score"):
        np.testing.assert_array_equal(r[k].numpy()[:nq], getattr(out, k).cpu().numpy()[:nq])


def test_repeat_calls_are_deterministic(E, ctx, heavy_parts):
    """Scratch counters/thresholds are reset between calls: identical outputs."""
    pool = workload.pool("heavy", 400_000, 308, shuffled=True)
    args = [torch.from_numpy(pool[k]).cuda() for k in ("len", "arrival", "cost")]
    outs = [gpu_result(E.tick(ctx, *args, to_gpu_partition(E, heavy_parts["quantile"]), E.meta(**THETA0),
                              E.select_params(k=64))) for _ in range(3)]
    for o in outs[1:]:
        for k in ("topk_id", "count", "head_id", "topk_score"):
            np.testing.assert_array_equal(o[k], outs[0][k])


@pytest.fixture(scope="module")
def ctx_full(E):
    return E.Context(0, max_pool=10_000_000, max_history=1_000_000, max_k=64)


@pytest.mark.parametrize("mode", [0, 1])
def test_tick_full_size_c3(E, orc, ctx_full, mode):
    """BASELINE config C3 at full size, in the launch configuration bench.py times:
    10M heavy-tailed pool, Refine-and-Prune partition of heavy(1M, seed 301), K=64.
    The oracle computes the whole tick, so every output is compared."""
    s, opart, _ = orc.partition(workload.heavy(1_000_000, 301))
    assert s == orc.OK
    pool = workload.pool("heavy", 10_000_000, 302)
    g, ref, phi = _run_both(E, orc, ctx_full, pool, opart, 64, mode)
    _check(g, ref, phi, pool, mode, 64)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", [0, 1])
def test_sharded_tick_records_on_one_gpu(E, orc, ctx, heavy_parts, world, mode):
    """The multi-GPU path with the all-gather replaced by a plain
    concatenation on one device: every shard runs ewsjf_tick_local (route + score
    + local top-K -> exchange record, global ids), the records of all shards are
    merged by ewsjf_tick_merge; the result equals the oracle tick over the whole
    pool (world-size invariance), qids of each shard included."""
    import torch
    pool = workload.pool("heavy", 300_001, 311)
    n = len(pool["len"])
    opart = heavy_parts["rp"]
    K = 32
    theta, sp = E.meta(**THETA0), E.select_params(k=K, mode=mode)
    dev = {k: torch.from_numpy(pool[k]).cuda() for k in ("len", "arrival", "cost")}
    qid = torch.full((n,), -7, dtype=torch.int32, device="cuda")
    recs, bounds = [], []
    for r in range(world):
        lo, hi = workload.shard_range(n, r, world)
        bounds.append((lo, hi))
        recs.append(E.tick_local(ctx, dev["len"][lo:hi], dev["arrival"][lo:hi], dev["cost"][lo:hi], lo,
                                 to_gpu_partition(E, opart), theta, sp, qid_out=qid[lo:hi]).clone())
    allx = torch.cat(recs)
    ref = orc.tick(pool["len"], pool["arrival"], pool["cost"], opart, orc.meta(**THETA0),
                   orc.select_params(k=K, mode=mode))
    phi, _ = orc.score_all(pool["len"], pool["arrival"], pool["cost"], ref["qid"], ref["partition"],
                           orc.meta(**THETA0), orc.select_params(k=K, mode=mode))
    for r, (lo, hi) in enumerate(bounds):      # every "rank" merges the same records
        gp = to_gpu_partition(E, opart)
        out = E.tick_merge(ctx, allx, world, lo, hi - lo, qid[lo:hi], gp, theta, sp)
        g = gpu_result(out)
        compare_selection(g, ref, phi, pool["arrival"], mode, K)
    np.testing.assert_array_equal(qid.cpu().numpy(), ref["qid"])


@pytest.mark.parametrize("mode", [0, 1])
def test_tick_full_size_with_holes(E, orc, ctx_full, mode):
    """App. D at pool scale: the C3 pool routed by the R&P partition with three of
    its queues removed (five ranges become holes holding >= 1% of the 10M
    requests).  Alg. 2 runs over every gap request in index order; qids, bubbles
    and every selection output equal the oracle's."""
    s, opart, _ = orc.partition(workload.heavy(1_000_000, 301))
    qs = opart.queues()
    keep = [q for i, q in enumerate(qs) if i not in (5, 11, 17, 23, len(qs) - 3)]
    hole = orc.make_partition([(q["min_len"], q["max_len"]) for q in keep], means=[q["mean"] for q in keep])
    pool = workload.pool("heavy", 10_000_000, 302)
    g, ref, phi = _run_both(E, orc, ctx_full, pool, hole, 64, mode)
    assert g["n_gap"] >= 100_000, g["n_gap"]
    _check(g, ref, phi, pool, mode, 64)


def test_sharded_tick_with_holes_at_pool_scale(E, orc, ctx_full):
    """App. D across shards: the 10M C3 pool with five hole
    ranges (>= 1% of the requests fall between queues), split over 2 simulated
    ranks whose exchange records carry all of their gap requests (the record's
    gap capacity raised with ewsjf_ctx_set_exchange_gap_cap).  The merge runs
    Alg. 2 over the union in global index order: qids, bubbles and selections
    equal the oracle's single-pool tick."""
    s, opart, _ = orc.partition(workload.heavy(1_000_000, 301))
    qs = opart.queues()
    keep = [q for i, q in enumerate(qs) if i not in (5, 11, 17, 23, len(qs) - 3)]
    hole = orc.make_partition([(q["min_len"], q["max_len"]) for q in keep], means=[q["mean"] for q in keep])
    pool = workload.pool("heavy", 10_000_000, 302)
    n, world, K, mode = len(pool["len"]), 2, 64, 0
    theta, sp = E.meta(**THETA0), E.select_params(k=K, mode=mode)
    dev = {k: torch.from_numpy(pool[k]).cuda() for k in ("len", "arrival", "cost")}
    qid = torch.full((n,), -7, dtype=torch.int32, device="cuda")
    small = E.exchange_bytes(ctx_full, hole.n, K)
    ctx_full.set_exchange_gap_cap(n // world + 1)
    try:
        assert E.exchange_bytes(ctx_full, hole.n, K) > small
        recs, bounds = [], []
        for r in range(world):
            lo, hi = workload.shard_range(n, r, world)
            bounds.append((lo, hi))
            recs.append(E.tick_local(ctx_full, dev["len"][lo:hi], dev["arrival"][lo:hi], dev["cost"][lo:hi], lo,
                                     to_gpu_partition(E, hole), theta, sp, qid_out=qid[lo:hi]).clone())
        allx = torch.cat(recs)
        ref = orc.tick(pool["len"], pool["arrival"], pool["cost"], hole, orc.meta(**THETA0),
                       orc.select_params(k=K, mode=mode))
        phi, _ = orc.score_all(pool["len"], pool["arrival"], pool["cost"], ref["qid"], ref["partition"],
                               orc.meta(**THETA0), orc.select_params(k=K, mode=mode))
        gs = []
        for r, (lo, hi) in enumerate(bounds):      # each rank finalises its own shard's gap qids
            gp = to_gpu_partition(E, hole)
            out = E.tick_merge(ctx_full, allx, world, lo, hi - lo, qid[lo:hi], gp, theta, sp)
            g = gpu_result(out)
            g["part"] = gp
            gs.append(g)
        full = qid.cpu().numpy()
        for g in gs:
            g["qid"] = full
            assert g["n_gap"] >= 100_000, g["n_gap"]
            _check(g, ref, phi, pool, mode, K)
    finally:
        ctx_full.set_exchange_gap_cap(1024)


@pytest.mark.parametrize("case", ["plain", "few_gaps", "many_gaps"])
def test_tick_host_pipelined_equals_device(E, orc, ctx_full, heavy_parts, case):
    """ewsjf_tick_host pipelines pools >= 2M (chunked H2D on one stream, per-chunk local
    ticks into exchange records, qid slices back on another stream, one merge): its
    results equal the single-pass device tick's.  few_gaps: a partition with one hole
    (Alg. 2 in the merge, the gap requests' qids re-read after it); many_gaps: holes
    holding more gap requests than an exchange record carries (the call redoes the tick
    in one pass over the pool already on the device)."""
    n = 3_000_000
    pool = workload.pool("heavy", n, 309)
    if case == "plain":
        part_o = heavy_parts["rp"]
    else:
        s, opart, _ = orc.partition(workload.heavy(1_000_000, 301))
        qs = opart.queues()
        bounds = [(q["min_len"], q["max_len"]) for q in qs]
        means = [q["mean"] for q in qs]
        if case == "few_gaps":
            # the last (long-prompt) queue split around a hole [20000, 20000 + w) holding a few
            # hundred of the pool's requests (Pareto tail: ~1.5 requests per length there)
            lo, hi = bounds[-1]
            w = 1
            while ((pool["len"] >= 20000) & (pool["len"] < 20000 + 2 * w)).sum() <= 600:
                w *= 2
            bounds[-1] = (lo, 20000)
            bounds.append((20000 + w, hi))
            means.append(means[-1])
        else:
            drop = (5, 11, 17, 23, len(qs) - 3)
            bounds = [b for i, b in enumerate(bounds) if i not in drop]
            means = [m for i, m in enumerate(means) if i not in drop]
        part_o = orc.make_partition(bounds, means=means)
    theta, sp = E.meta(**THETA0), E.select_params(k=64)
    hl, ha, hc = (torch.from_numpy(pool[k]).pin_memory() for k in ("len", "arrival", "cost"))
    hq = torch.full((n,), -7, dtype=torch.int32).pin_memory()
    gp_host, gp_dev = to_gpu_partition(E, part_o), to_gpu_partition(E, part_o)
    r = E.tick_host(ctx_full, hl, ha, hc, gp_host, theta, sp, qid_out=hq)
    dq = torch.empty(n, dtype=torch.int32, device="cuda")
    out = E.tick(ctx_full, hl.cuda(), ha.cuda(), hc.cuda(), gp_dev, theta, sp, qid_out=dq)
    if case == "few_gaps":
        assert 0 < out.summary["n_gap"] <= 1024, out.summary["n_gap"]
    if case == "many_gaps":
        assert out.summary["n_gap"] > 3 * 1024, out.summary["n_gap"]
    assert r["summary"] == out.summary
    np.testing.assert_array_equal(hq.numpy(), dq.cpu().numpy())
    assert [(q.min_len, q.max_len, q.id) for q in gp_host.q[: gp_host.n]] == \
           [(q.min_len, q.max_len, q.id) for q in gp_dev.q[: gp_dev.n]]
    nq = out.summary["n_queues"]
    for k in ("topk_id", "count", "head_id", "topk_score", "head_score", "max_score"):
        np.testing.assert_array_equal(r[k].numpy()[:nq], getattr(out, k).cpu().numpy()[:nq])
