"""GPU parity of Alg. 1's Batch Builder (ewsjf_batch_build)
against the oracle's O12 (oracle.batch): FIFO tick on the GPU -> batch kernel,
versus oracle tick (primary) -> oracle.batch over the same routed pool.  Batch
ids (in admission order), token totals and the primary are compared exactly."""
import numpy as np
import pytest
import torch

import workload
from tests.parity import to_gpu_partition

pytestmark = pytest.mark.gpu

THETA0 = workload.THETA0


@pytest.fixture(scope="module")
def E():
    import paper_2601_21758_b200 as E
    return E


@pytest.fixture(scope="module")
def ctx(E):
    return E.Context(0, max_pool=1 << 22, max_history=1 << 21, max_k=256)


@pytest.fixture(scope="module")
def part_c1(orc):
    s, part, _ = orc.partition(workload.bimodal(10_000, 101), merge_rule=orc.MAX_U)
    assert s == orc.OK
    return part


def _both(E, orc, ctx, pool, opart, max_req, max_tok, K=None, now=600.0, base=0):
    K = K or max_req
    n = len(pool["len"])
    ln = torch.from_numpy(pool["len"]).cuda()
    ar = torch.from_numpy(pool["arrival"]).cuda()
    co = torch.from_numpy(pool["cost"]).cuda() if pool["cost"] is not None else None
    gpart = to_gpu_partition(E, opart)
    out = E.tick(ctx, ln, ar, co, gpart, E.meta(**THETA0), E.select_params(k=K, mode=1, now=now),
                 global_base=base)
    ids, info = E.batch_build(ctx, ln, out, out.summary["n_queues"], max_req, max_tok, global_base=base)
    torch.cuda.synchronize()
    info = info.cpu().numpy()
    ids = ids.cpu().numpy()
    sp = orc.select_params(k=K, mode=1, now=now)
    ref = orc.tick(pool["len"], pool["arrival"], pool["cost"], opart, orc.meta(**THETA0), sp, global_base=base)
    rid, rtok = orc.batch(pool["len"], pool["arrival"], pool["cost"], ref["qid"], ref["partition"], sp,
                          ref["primary"], max_req, max_tok, global_base=base)
    assert info[2] == 0, "device status"
    assert info[3] == ref["primary"] == out.summary["primary"]
    assert info[0] == len(rid) and info[1] == rtok
    np.testing.assert_array_equal(ids[: info[0]], rid)
    assert (ids[info[0]:] == -1).all()
    return rid, rtok


@pytest.mark.parametrize("max_req,max_tok", [(1, 1), (8, 4096), (64, 16384), (64, 1 << 30), (256, 65536),
                                             (33, 2000)])
def test_batch_matches_oracle_c1(E, orc, ctx, part_c1, max_req, max_tok):
    pool = workload.pool("bimodal", 3000, 311)
    _both(E, orc, ctx, pool, part_c1, max_req, max_tok)


def test_batch_backfill_spans_queues(E, orc, ctx):
    """Tiny queues around the primary: the batch crosses several neighbours (R29)."""
    opart = orc.make_partition([(1, 16), (16, 64), (64, 256), (256, 1024), (1024, 4096), (4096, 16385)])
    pool = workload.pool("heavy", 200, 77)
    rid, _ = _both(E, orc, ctx, pool, opart, 128, 1 << 20)
    assert len(rid) > 50


@pytest.mark.parametrize("seed", range(6))
def test_batch_random_budgets(E, orc, ctx, part_c1, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 5000))
    pool = workload.pool("bimodal" if seed % 2 else "heavy", n, 900 + seed)
    mr = int(rng.integers(1, 200)); mt = int(rng.integers(0, 200_000))
    _both(E, orc, ctx, pool, part_c1, mr, mt, K=int(rng.integers(mr, 257)), base=int(rng.integers(0, 1 << 31)))


def test_batch_empty_pool_and_oversized_first(E, orc, ctx, part_c1):
    pool = workload.pool("bimodal", 1, 5)
    rid, tok = _both(E, orc, ctx, pool, part_c1, 16, 0)       # first request admitted, over budget
    assert len(rid) == 1 and tok == pool["len"][0]
    pool = {"len": np.zeros(0, np.int32), "arrival": np.zeros(0, np.float32), "cost": np.zeros(0, np.float32)}
    rid, tok = _both(E, orc, ctx, pool, part_c1, 16, 100)
    assert len(rid) == 0 and tok == 0


def test_batch_full_size_c3(E, orc, ctx):
    """C3 shape (10M pending, bimodal): batch 256 / 64k tokens on the GPU; the oracle
    batch over the same routed pool is exact (it is O(n log n))."""
    s, opart, _ = orc.partition(workload.bimodal(200_000, 7), merge_rule=orc.MAX_U)
    big = E.Context(0, max_pool=10_000_000, max_history=1 << 20, max_k=256)
    pool = workload.pool("bimodal", 10_000_000, 8)
    _both(E, orc, big, pool, opart, 256, 65536)


def test_batch_rejects_shallow_rows(E, ctx, part_c1):
    pool = workload.pool("bimodal", 100, 1)
    ln = torch.from_numpy(pool["len"]).cuda()
    ar = torch.from_numpy(pool["arrival"]).cuda()
    gpart = to_gpu_partition(E, part_c1)
    out = E.tick(ctx, ln, ar, None, gpart, E.meta(**THETA0), E.select_params(k=8, mode=1, now=600.0))
    with pytest.raises(Exception):
        E.batch_build(ctx, ln, out, out.summary["n_queues"], 16, 1000)


def test_batch_many_queues_global_scratch(E, orc, ctx):
    """250 queues x 256-deep rows: the prefix table (256 KB) exceeds shared memory
    and lives in global scratch."""
    opart = orc.make_partition([(1 + 4 * i, 5 + 4 * i) for i in range(250)])
    rng = np.random.default_rng(4)
    n = 20_000
    ln = rng.integers(1, 1001, n).astype(np.int32)
    pool = {"len": ln, "arrival": workload.arrivals(n, 41), "cost": workload.cost_estimates(ln, 42)}
    for mr, mt in [(256, 1 << 20), (256, 3000), (200, 50_000)]:
        _both(E, orc, ctx, pool, opart, mr, mt)
