"""The product's sharded tick across real processes: two ranks on the
one GPU of the test box, each running the library's ewsjf_tick_local on its
index shard of the pool; the rank records (the library's own exchange format)
are all-gathered over torch.distributed (gloo: NCCL needs one device per rank)
and every rank runs ewsjf_tick_merge on the gathered bytes.  Both ranks must
return the oracle's tick over the whole pool (replication, world-size
invariance), gap requests and bubbles included."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workload

pytestmark = pytest.mark.gpu

N = 120_001
K = 32


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


BOUNDS = [(32, 100), (100, 2001), (2001, 5000), (6200, 40000)]     # [5000, 6200) is a hole; 5501..5579 make bubbles


def _worker(rank, world, port, mode, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2601_21758_b200 as E
    torch.cuda.set_device(0)
    pool = workload.pool("heavy", N, 61)
    lo, hi = workload.shard_range(N, rank, world)
    dev = torch.device("cuda", 0)
    t = {k: torch.from_numpy(pool[k][lo:hi].copy()).to(dev) for k in ("len", "arrival", "cost")}
    ctx = E.Context(0, max_pool=N, max_history=0, max_k=64)
    th, sp = E.meta(**workload.THETA0), E.select_params(k=K, mode=mode)
    qid = torch.full((hi - lo,), -7, dtype=torch.int32, device=dev)
    rec = E.tick_local(ctx, t["len"], t["arrival"], t["cost"], lo, E.make_partition(BOUNDS), th, sp, qid_out=qid)
    torch.cuda.synchronize()
    mine = rec.cpu()
    allrec = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allrec, mine)                    # the product's exchange bytes cross the collective
    allx = torch.cat(allrec).to(dev)
    part = E.make_partition(BOUNDS)
    res = E.tick_merge(ctx, allx, world, lo, hi - lo, qid, part, th, sp)
    g = {k: getattr(res, k).cpu().numpy() for k in ("topk_id", "topk_score", "count", "head_id", "head_score",
                                                   "max_score")}
    g.update(res.summary)
    g["qid"] = qid.cpu().numpy()
    g["bounds"] = [(q["min_len"], q["max_len"]) for q in part.queues()]
    out[rank] = g
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [0, 1])
def test_two_rank_tick_over_gloo_matches_oracle(orc, mode):
    from tests.parity import compare_selection
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), mode, out), nprocs=world, join=True)
    pool = workload.pool("heavy", N, 61)
    opart = orc.make_partition(BOUNDS)
    ref = orc.tick(pool["len"], pool["arrival"], pool["cost"], opart, orc.meta(**workload.THETA0),
                   orc.select_params(k=K, mode=mode))
    phi, _ = orc.score_all(pool["len"], pool["arrival"], pool["cost"], ref["qid"], ref["partition"],
                           orc.meta(**workload.THETA0), orc.select_params(k=K, mode=mode))
    assert ref["n_bubbles"] > 0
    qid = np.concatenate([out[r]["qid"] for r in range(world)])
    np.testing.assert_array_equal(qid, ref["qid"])
    for r in range(world):
        assert out[r]["bounds"] == [(q["min_len"], q["max_len"]) for q in ref["partition"].queues()]
        compare_selection(out[r], ref, phi, pool["arrival"], mode, K)
