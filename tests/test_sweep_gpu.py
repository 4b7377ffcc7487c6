"""GPU parity of the Θ sweep (A12, config C5; §4.4.2) against the
CPU oracle's O11, and self-consistency with independent score_select calls.

Snapshot = bimodal pool routed by the Refine-and-Prune partition of a bimodal
history (C2's partition), Θ uniform in S:500's bounds.
"""
import numpy as np
import pytest
import torch

import workload
from tests.parity import compare_selection, gpu_result, to_gpu_partition

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import paper_2601_21758_b200 as E
    return E


@pytest.fixture(scope="module")
def ctx(E):
    return E.Context(0, max_pool=1 << 21, max_history=0, max_k=64, max_sweep=1 << 21)


@pytest.fixture(scope="module")
def c2_partition(orc):
    s, part, _ = orc.partition(workload.bimodal(1_000_000, 201))
    assert s == orc.OK
    return part


def _snapshot(orc, opart, n, seed):
    pool = workload.pool("bimodal", n, seed)
    s, qid, *_ = orc.route(pool["len"], orc.copy_partition(opart), 64)
    assert s == orc.OK      # the snapshot is routed by the same partition: no bubbles
    return pool, qid


def _run_sweep(E, ctx, pool, qid, opart, thetas, K, mode):
    dev = [torch.from_numpy(pool[k]).cuda() for k in ("len", "arrival", "cost")] + [torch.from_numpy(qid).cuda()]
    outs = E.score_select_sweep(ctx, *dev, to_gpu_partition(E, opart), [E.meta(**t) for t in thetas],
                                E.select_params(k=K, mode=mode))
    torch.cuda.synchronize()
    res = []
    for o in outs:
        o.fetch_summary()
        res.append(gpu_result(o))
    return res, dev


def _check_against_oracle(orc, pool, qid, opart, thetas, res, K, mode):
    sp = orc.select_params(k=K, mode=mode)
    st, ref = orc.sweep(pool["len"], pool["arrival"], pool["cost"], qid, opart, thetas, sp)
    assert len(ref) == len(res)
    for t, (g, r) in enumerate(zip(res, ref)):
        phi, _ = orc.score_all(pool["len"], pool["arrival"], pool["cost"], qid, opart, orc.meta(**thetas[t]), sp)
        compare_selection(g, r, phi, pool["arrival"], mode, K)


@pytest.mark.parametrize("K", [1, 16, 64])
def test_sweep_matches_oracle(E, orc, ctx, c2_partition, K):
    pool, qid = _snapshot(orc, c2_partition, 200_003, 501)
    thetas = workload.random_thetas(12, 502)
    res, _ = _run_sweep(E, ctx, pool, qid, c2_partition, thetas, K, 0)
    _check_against_oracle(orc, pool, qid, c2_partition, thetas, res, K, 0)


def test_sweep_rejects_fifo_mode(E, orc, ctx, c2_partition):
    pool, qid = _snapshot(orc, c2_partition, 1000, 505)
    with pytest.raises(E.EwsjfError):
        _run_sweep(E, ctx, pool, qid, c2_partition, workload.random_thetas(2, 1), 4, 1)


def test_sweep_batch_invariance(E, orc, ctx, c2_partition):
    """A12 = n_Θ independent A11 runs (SURVEY §8c pin): Θ_t's result does not depend
    on the other Θ of the sweep (bit for bit), and equals the oracle's O11."""
    pool, qid = _snapshot(orc, c2_partition, 150_000, 503)
    thetas = workload.random_thetas(19, 504)
    res, dev = _run_sweep(E, ctx, pool, qid, c2_partition, thetas, 16, 0)
    for t in (0, 7, 18):
        one, _ = _run_sweep(E, ctx, pool, qid, c2_partition, [thetas[t]], 16, 0)
        one = one[0]
        nq = one["n_queues"]
        assert res[t]["n_queues"] == nq and res[t]["primary"] == one["primary"]
        for k in ("topk_id", "topk_score", "count", "head_id", "head_score", "max_score"):   # rows >= nq unused
            np.testing.assert_array_equal(res[t][k][:nq], one[k][:nq], err_msg=f"theta {t} {k}")
    _check_against_oracle(orc, pool, qid, c2_partition, thetas, res, 16, 0)


def test_sweep_more_than_one_batch_and_deep_k(E, orc, ctx, c2_partition):
    """n_Θ above the kernel batch (128) and K above the register-selection limit
    (the score_select path) both match the oracle."""
    pool, qid = _snapshot(orc, c2_partition, 20_000, 506)
    thetas = workload.random_thetas(131, 507)
    res, _ = _run_sweep(E, ctx, pool, qid, c2_partition, thetas, 8, 0)
    _check_against_oracle(orc, pool, qid, c2_partition, thetas[120:], res[120:], 8, 0)
    res, _ = _run_sweep(E, ctx, pool, qid, c2_partition, thetas[:3], 64, 0)
    _check_against_oracle(orc, pool, qid, c2_partition, thetas[:3], res, 64, 0)


def test_sweep_edge_cases(E, orc, ctx):
    """Empty queues, invalid / excluded requests, K above every queue's size."""
    part = orc.make_partition([(1, 50), (50, 100), (100, 200), (200, 400)])
    rng = np.random.default_rng(9)
    n = 3000
    lens = rng.integers(1, 200, size=n).astype(np.int32)        # queue 3 stays empty
    arr = np.sort(rng.random(n) * 500).astype(np.float32)
    arr[::97] = 700.0                                             # arrival > now: excluded
    cost = workload.cost_estimates(lens, 9)
    cost[::89] = -1.0                                             # C <= 0: excluded
    s, qid, *_ = orc.route(lens, orc.copy_partition(part), 64)
    qid[::101] = 77                                               # unknown queue id: invalid
    pool = {"len": lens, "arrival": arr, "cost": cost}
    thetas = workload.random_thetas(5, 8)
    res, _ = _run_sweep(E, ctx, pool, qid, part, thetas, 40, 0)
    _check_against_oracle(orc, pool, qid, part, thetas, res, 40, 0)
    st, ref = orc.sweep(lens, arr, cost, qid, part, thetas, orc.select_params(k=40))
    for g, r in zip(res, ref):
        assert g["n_invalid"] == r["n_invalid"] and g["n_excluded"] == r["n_excluded"]
        assert g["primary"] == r["primary"]


def test_sweep_full_size_c5(E, orc, ctx, c2_partition):
    """BASELINE C5 at full size in bench.py's launch configuration: all 256 Θ over
    the 1M bimodal snapshot routed by the C2 partition in ONE call, K=16; a strided
    subset of 24 Θ is checked against the oracle (its full sort per Θ is slow)."""
    pool, qid = _snapshot(orc, c2_partition, 1_000_000, 501)
    thetas = workload.random_thetas(256, 502)
    res, _ = _run_sweep(E, ctx, pool, qid, c2_partition, thetas, 16, 0)
    _check_against_oracle(orc, pool, qid, c2_partition, thetas[::11], res[::11], 16, 0)


@pytest.mark.parametrize("kind", ["bimodal", "heavy"])
def test_sweep_prefilter_matches_full_evaluation(E, orc, ctx, c2_partition, kind, monkeypatch):
    """The Θ-independent dominance prefilter (sweep.cu K3a-K3g) against the sweep
    without it (EWSJF_NO_SKY) and against the oracle: lengths 1 (where
    ln(b+1)/(b+1) still rises), lengths past the 65536 grouping range, ties."""
    rng = np.random.default_rng(12 if kind == "heavy" else 13)
    n = 60_000
    lens = workload.lengths(kind, n, 14).copy()
    lens[rng.integers(0, n, 300)] = 1
    lens[rng.integers(0, n, 300)] = 2
    lens[rng.integers(0, n, 200)] = 70_000 + rng.integers(0, 500, 200)
    part = orc.make_partition([(1, 3), (3, 64), (64, 3000), (3000, 71_000)])
    arr = workload.arrivals(n, 15)
    arr[::50] = arr[0]                                        # exact feature ties across ids
    cost = workload.cost_estimates(lens, 16)
    s, qid, *_ = orc.route(lens, orc.copy_partition(part), 64)
    pool = {"len": lens, "arrival": arr, "cost": cost}
    thetas = workload.random_thetas(9, 17) + [dict(a_b=0.0, b_b=1.0, a_u=0.0, b_u=0.0, a_f=0.0, b_f=0.0),
                                              dict(a_b=0.0, b_b=0.0, a_u=0.0, b_u=0.0, a_f=0.0, b_f=2.0)]
    res, _ = _run_sweep(E, ctx, pool, qid, part, thetas, 16, 0)
    _check_against_oracle(orc, pool, qid, part, thetas, res, 16, 0)
    monkeypatch.setenv("EWSJF_NO_SKY", "1")
    full, _ = _run_sweep(E, ctx, pool, qid, part, thetas, 16, 0)
    for a, b in zip(res, full):
        nq = a["n_queues"]
        np.testing.assert_array_equal(a["count"][:nq], b["count"][:nq])
        np.testing.assert_array_equal(a["head_id"][:nq], b["head_id"][:nq])
        np.testing.assert_array_equal(a["topk_id"][:nq], b["topk_id"][:nq])      # same fp32 keys: identical
