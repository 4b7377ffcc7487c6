"""Host half of Alg. 1 (lines 8-12): ewsjf_prune_empty in libewsjf against the
oracle's or_prune_empty on random counter states (no GPU needed: the call is
host bookkeeping over the host partition)."""
import numpy as np
import pytest

from tests.parity import to_gpu_partition


@pytest.fixture(scope="module")
def E():
    import paper_2601_21758_b200 as E
    return E


@pytest.mark.parametrize("seed", range(20))
def test_prune_empty_matches_oracle(E, orc, seed):
    rng = np.random.default_rng(seed)
    nq = int(rng.integers(1, 40))
    edges = np.sort(rng.choice(np.arange(2, 5000), nq - 1, replace=False)) if nq > 1 else np.array([], int)
    b = [1] + [int(x) for x in edges] + [5001]
    opart = orc.make_partition([(b[i], b[i + 1]) for i in range(nq)])
    e0 = rng.integers(0, 6, nq).astype(np.int32)
    counts = np.where(rng.random(nq) < 0.5, 0, rng.integers(1, 100, nq)).astype(np.int64)
    thr = int(rng.integers(0, 6))
    gp = to_gpu_partition(E, opart)
    for i in range(nq):
        gp.q[i].empty_count = int(e0[i])
    v0 = gp.version
    rm = E.prune_empty(gp, counts, thr)
    op, oe, orm = orc.prune_empty(opart, e0, counts, thr)
    assert rm == orm and gp.n == op.n
    assert [(q["min_len"], q["max_len"], q["id"], q["index"]) for q in gp.queues()] == \
           [(q["min_len"], q["max_len"], q["id"], q["index"]) for q in op.queues()]
    assert [gp.q[i].empty_count for i in range(gp.n)] == list(oe)
    assert gp.version == v0 + (1 if rm else 0)


def test_prune_empty_alternating_queue_is_never_removed(E, orc):
    """empty_count counts CONSECUTIVE empty tactical steps ("remain empty"):
    a queue empty on every other tick never exceeds 1 and is never removed, in both the
    library and the oracle, while a queue that stays empty goes once its counter passes
    the threshold (strict, R25)."""
    opart = orc.make_partition([(1, 10), (10, 20), (20, 30)])
    gp = to_gpu_partition(E, opart)
    oe = np.zeros(3, dtype=np.int32)
    op = opart
    for tick in range(12):
        counts = np.array([5, 0 if tick % 2 == 0 else 3, 0 if tick < 11 else 0], dtype=np.int64)[: gp.n]
        if gp.n == 2:
            counts = counts[:2]
        E.prune_empty(gp, counts, 2)
        op, oe, _ = orc.prune_empty(op, oe, counts, 2)
        assert [q["id"] for q in gp.queues()] == [q["id"] for q in op.queues()]
        assert [gp.q[i].empty_count for i in range(gp.n)] == list(oe)
        assert 1 in [q["id"] for q in gp.queues()]          # the alternating queue stays
    assert [q["id"] for q in gp.queues()] == [0, 1]          # the always-empty queue is gone
