"""World-size-2/3 gloo tests of the sharded tick protocol on CPU.

Each rank owns the index range [floor(rN/P), floor((r+1)N/P)) of the pool,
reduces it to a fixed-size exchange record keyed by GLOBAL ids (here computed
by the oracle — the CUDA kernels need a GPU), the records are all-gathered over
torch.distributed (gloo here, NCCL on the GPU box) and every rank merges them.
The merged result must equal the single-process oracle tick over the whole pool
on every rank (world-size invariance, replication), including gap requests,
which are exchanged and run through Alg. 2 in global index order (R22)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workload

K = 16
N = 6000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partition(O, holes: bool):
    if holes:
        return O.make_partition([(32, 100), (180, 300), (1000, 2000)], means=[60, 240, 1500])
    return O.make_partition(workload.quantile_bounds(workload.heavy(50_000, 9), 8))


def _record(O, pool, lo, hi, part, mode):
    """Rank-local exchange record: per queue top-K (gid, score, key) + count + head."""
    sp = O.select_params(k=K, mode=mode)
    th = O.meta(**workload.THETA0)
    lens = pool["len"][lo:hi]
    # gap requests are not routed locally: they travel in the record (gid, len, arrival, cost)
    p2 = O.copy_partition(part)
    bounds = [(q["min_len"], q["max_len"]) for q in part.queues()]
    ing = np.array([not any(a <= b < c for a, c in bounds) and b >= 1 for b in lens])
    keep = ~ing
    res = O.tick(np.where(keep, lens, 0), pool["arrival"][lo:hi], pool["cost"][lo:hi], p2, th, sp, global_base=lo)
    rec = np.zeros((part.n, K, 3), np.float64)
    for p in range(part.n):
        rec[p, :, 0] = res["topk_id"][p]
        rec[p, :, 1] = res["topk_score"][p]
        ids = res["topk_id"][p]
        rec[p, :, 2] = [pool["arrival"][i] if i >= 0 else np.inf for i in ids]
    meta = np.zeros((part.n, 4), np.float64)
    meta[:, 0] = res["count"][: part.n]
    meta[:, 1] = res["head_id"][: part.n]
    meta[:, 2] = [pool["arrival"][h] if h >= 0 else np.inf for h in res["head_id"][: part.n]]
    meta[:, 3] = res["head_score"][: part.n]
    gap = np.nonzero(ing)[0] + lo
    return rec, meta, gap


def _worker(rank, world, port, holes, mode, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    pool = workload.pool("heavy", N, 77)
    if holes:
        pool["len"] = np.random.default_rng(5).integers(1, 4000, size=N).astype(np.int32)
    part = _partition(O, holes)
    lo, hi = workload.shard_range(N, rank, world)
    rec, meta, gap = _record(O, pool, lo, hi, part, mode)
    # fixed-size records -> all_gather (the NCCL allgather of tick_sharded)
    t_rec = torch.from_numpy(rec.reshape(-1))
    t_meta = torch.from_numpy(meta.reshape(-1))
    g_rec = [torch.empty_like(t_rec) for _ in range(world)]
    g_meta = [torch.empty_like(t_meta) for _ in range(world)]
    dist.all_gather(g_rec, t_rec)
    dist.all_gather(g_meta, t_meta)
    cnt = torch.tensor([len(gap)], dtype=torch.int64)
    g_cnt = [torch.empty_like(cnt) for _ in range(world)]
    dist.all_gather(g_cnt, cnt)
    cap = int(max(c.item() for c in g_cnt))
    t_gap = torch.full((cap,), -1, dtype=torch.int64)
    t_gap[: len(gap)] = torch.from_numpy(gap)
    g_gap = [torch.empty_like(t_gap) for _ in range(world)]
    dist.all_gather(g_gap, t_gap)
    # replicated merge on every rank
    nq = part.n
    recs = [g.numpy().reshape(nq, K, 3) for g in g_rec]
    metas = [g.numpy().reshape(nq, 4) for g in g_meta]
    merged = {"count": [], "head_id": [], "topk_id": []}
    for p in range(nq):
        cand = [(r[p, j, 1], -r[p, j, 0], r[p, j, 2]) for r in recs for j in range(K) if r[p, j, 0] >= 0]
        if mode == 0:
            cand.sort(key=lambda x: (-x[0], -x[1]))
        else:
            cand.sort(key=lambda x: (x[2], -x[1]))
        merged["topk_id"].append([int(-c[1]) for c in cand[:K]] + [-1] * (K - min(K, len(cand))))
        merged["count"].append(int(sum(m[p, 0] for m in metas)))
        heads = [(m[p, 2], m[p, 1]) for m in metas if m[p, 1] >= 0]
        merged["head_id"].append(int(min(heads)[1]) if heads else -1)
    # gap requests of all ranks, in GLOBAL index order, through Alg. 2
    all_gap = np.sort(np.concatenate([g.numpy()[g.numpy() >= 0] for g in g_gap]))
    p2 = O.copy_partition(part)
    s, gq, *_ = O.route(pool["len"][all_gap], p2, 64)
    out[rank] = {"merged": merged, "gap_qid": gq.tolist(), "bounds": [(q["min_len"], q["max_len"]) for q in p2.queues()]}
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", [0, 1])
def test_sharded_merge_equals_single_process(orc, world, mode):
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), False, mode, out), nprocs=world, join=True)
    pool = workload.pool("heavy", N, 77)
    part = _partition(orc, False)
    ref = orc.tick(pool["len"], pool["arrival"], pool["cost"], part, orc.meta(**workload.THETA0),
                   orc.select_params(k=K, mode=mode))
    for r in range(world):
        m = out[r]["merged"]
        assert m == out[0]["merged"]                               # replicated
        assert m["count"] == ref["count"][: part.n].tolist()
        assert m["head_id"] == ref["head_id"][: part.n].tolist()
        assert m["topk_id"] == ref["topk_id"][: part.n].tolist()  # world-size invariant


def test_sharded_gap_requests_make_bubbles_in_global_order(orc):
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), True, 0, out), nprocs=2, join=True)
    pool_len = np.random.default_rng(5).integers(1, 4000, size=N).astype(np.int32)
    part = _partition(orc, True)
    p2 = orc.copy_partition(part)
    s, qid, *_ = orc.route(pool_len, p2, 64)
    ref_bounds = [(q["min_len"], q["max_len"]) for q in p2.queues()]
    assert out[0]["bounds"] == out[1]["bounds"] == ref_bounds
    bounds = [(q["min_len"], q["max_len"]) for q in part.queues()]
    gap_idx = [i for i, b in enumerate(pool_len) if b >= 1 and not any(a <= b < c for a, c in bounds)]
    assert out[0]["gap_qid"] == qid[gap_idx].tolist()
