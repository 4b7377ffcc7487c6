"""GPU parity of the online adjust mode (ewsjf_online_adjust, SURVEY §8f rank 3,
reading R31) against the oracle's O13: moved boundaries are compared exactly."""
import numpy as np
import pytest
import torch

import workload
from tests.parity import to_gpu_partition

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import paper_2601_21758_b200 as E
    return E


@pytest.fixture(scope="module")
def ctx(E):
    return E.Context(0, max_pool=1024, max_history=1 << 22, max_k=8)


def _both(E, orc, ctx, opart, window, s):
    gp = to_gpu_partition(E, opart)
    mv = E.online_adjust(ctx, torch.from_numpy(np.ascontiguousarray(window, np.int32)).cuda(), gp, s)
    op, omv = orc.online_adjust(np.asarray(window, np.int32), opart, s)
    assert mv == omv
    assert [(q["min_len"], q["max_len"], q["id"]) for q in gp.queues()] == \
           [(q["min_len"], q["max_len"], q["id"]) for q in op.queues()]
    return gp


@pytest.mark.parametrize("s", [0.0, 0.1, 0.25, 0.49])
@pytest.mark.parametrize("kind,seed", [("heavy", 1), ("bimodal", 2)])
def test_online_adjust_rp_partition(E, orc, ctx, s, kind, seed):
    """Refine-and-Prune partition of a history, window from a different seed and
    from the other distribution (large shifts, clamped)."""
    st_, opart, _ = orc.partition(workload.lengths(kind, 100_000, seed), merge_rule=orc.MAX_U)
    for wk in ("heavy", "bimodal"):
        _both(E, orc, ctx, opart, workload.lengths(wk, 200_000, seed + 10), s)


@pytest.mark.parametrize("seed", range(12))
def test_online_adjust_random(E, orc, ctx, seed):
    rng = np.random.default_rng(seed)
    nq = int(rng.integers(2, 40))
    edges = np.sort(rng.choice(np.arange(2, 30_000), nq - 1, replace=False))
    b = [1] + [int(x) for x in edges] + [30_001]
    opart = orc.make_partition([(b[i], b[i + 1]) for i in range(nq)])
    for i in range(nq):
        opart.q[i].count = int(rng.integers(0, 1000)) if rng.random() > 0.1 else 0
    window = rng.integers(-5, 31_000, int(rng.integers(0, 50_000))).astype(np.int32)
    _both(E, orc, ctx, opart, window, float(rng.choice([0.0, 0.25, 0.3, 0.45])))


def test_online_adjust_window_in_one_queue_and_empty(E, orc, ctx):
    opart = orc.make_partition([(1, 10), (10, 20), (20, 30)])
    for i in range(3):
        opart.q[i].count = 10
    gp = _both(E, orc, ctx, opart, [12, 12, 12, 12], 0.25)
    assert [(q["min_len"], q["max_len"]) for q in gp.queues()] == [(1, 12), (12, 18), (18, 30)]
    _both(E, orc, ctx, opart, np.zeros(0, np.int32), 0.25)
    with pytest.raises(Exception):
        E.online_adjust(ctx, torch.tensor([5], dtype=torch.int32, device="cuda"), to_gpu_partition(E, opart), 0.5)
