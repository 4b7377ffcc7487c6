"""The index-sharded tick through the library's own NCCL communicator
(ewsjf_ctx_init_nccl): local route+score+reduce -> ncclAllGather
on the ctx stream -> merge, all inside ewsjf_tick.  On one GPU the world is 1;
the result must equal the oracle (and the single-GPU tick) exactly, also when
the three steps are replayed from a CUDA graph."""
import numpy as np
import pytest
import torch

import oracle as O
import workload
from tests.parity import compare_selection, gpu_result, to_gpu_partition

pytestmark = pytest.mark.gpu


def _setup(n, seed, kind="heavy"):
    import paper_2601_21758_b200 as E
    hist = workload.lengths(kind, 50_000, seed)
    s, opart, _ = O.partition(hist)
    pool = workload.pool(kind, n, seed + 1)
    dev = torch.device("cuda", 0)
    t = {k: torch.from_numpy(pool[k]).to(dev) for k in ("len", "arrival", "cost")}
    return E, opart, pool, t, dev


@pytest.mark.parametrize("mode,k", [(0, 64), (1, 64), (0, 1), (1, 256)])
def test_nccl_world1_tick_matches_oracle(mode, k):
    E, opart, pool, t, dev = _setup(300_001, 41)
    ctx = E.Context(0, max_pool=1 << 20, max_history=0, max_k=256)
    ctx.init_nccl(0, 1)
    qid = torch.empty_like(t["len"])
    th = E.meta(**workload.THETA0)
    out = E.tick(ctx, t["len"], t["arrival"], t["cost"], to_gpu_partition(E, opart), th,
                 E.select_params(k=k, mode=mode), qid_out=qid)
    ref = O.tick(pool["len"], pool["arrival"], pool["cost"], opart, O.meta(**workload.THETA0),
                 O.select_params(k=k, mode=mode))
    phi, _ = O.score_all(pool["len"], pool["arrival"], pool["cost"], ref["qid"], ref["partition"],
                         O.meta(**workload.THETA0), O.select_params(k=k, mode=mode))
    np.testing.assert_array_equal(qid.cpu().numpy(), ref["qid"])
    compare_selection(gpu_result(out), ref, phi, pool["arrival"], mode, k)
    ctx.close()


def test_nccl_world1_gap_requests_and_graph_replay():
    """Gap-falling lengths (App. D, Alg. 2) through the exchange + NCCL path, and
    the whole sharded tick captured once in a CUDA graph and replayed."""
    import paper_2601_21758_b200 as E
    dev = torch.device("cuda", 0)
    bounds = [(32, 100), (100, 2001), (2001, 5000), (7000, 40000)]   # 5501..6299 make bubbles (Alg. 2)
    gp = E.make_partition(bounds)
    op = O.make_partition(bounds)
    pool = workload.pool("heavy", 30_000, 77)
    t = {k: torch.from_numpy(pool[k]).to(dev) for k in ("len", "arrival", "cost")}
    th = E.meta(**workload.THETA0)
    sp = E.select_params(k=32, mode=0)
    ctx = E.Context(0, max_pool=1 << 18, max_history=0, max_k=64)
    ctx.init_nccl(0, 1)
    qid = torch.empty_like(t["len"])
    out = E.tick(ctx, t["len"], t["arrival"], t["cost"], gp, th, sp, qid_out=qid)
    ref = O.tick(pool["len"], pool["arrival"], pool["cost"], op, O.meta(**workload.THETA0),
                 O.select_params(k=32, mode=0))
    np.testing.assert_array_equal(qid.cpu().numpy(), ref["qid"])
    phi, _ = O.score_all(pool["len"], pool["arrival"], pool["cost"], ref["qid"], ref["partition"],
                         O.meta(**workload.THETA0), O.select_params(k=32, mode=0))
    compare_selection(gpu_result(out), ref, phi, pool["arrival"], 0, 32)
    assert out.summary["n_queues"] == ref["nq"] > len(bounds)      # bubbles were created
    # graph: the partition with its bubbles is now stable (published), replay the tick
    gp2 = E.make_partition(bounds)
    out2 = E.Outputs.alloc(32, dev)
    E.tick(ctx, t["len"], t["arrival"], t["cost"], gp2, th, sp, qid_out=qid, out=out2)  # warm (LUT cached)
    gp3 = E.make_partition(bounds)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            E.tick(ctx, t["len"], t["arrival"], t["cost"], gp3, th, sp, qid_out=qid, out=out2, sync=False)
    torch.cuda.current_stream().wait_stream(s)
    for c in (out2.topk_id, out2.count, out2.head_id):
        c.zero_()
    qid.fill_(-7)
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(qid.cpu().numpy(), ref["qid"])
    nq = out.summary["n_queues"]            # rows past nq are not written
    np.testing.assert_array_equal(out2.count.cpu().numpy()[:nq], out.count.cpu().numpy()[:nq])
    np.testing.assert_array_equal(out2.topk_id.cpu().numpy()[:nq], out.topk_id.cpu().numpy()[:nq])
    np.testing.assert_array_equal(out2.head_id.cpu().numpy()[:nq], out.head_id.cpu().numpy()[:nq])
    ctx.detach_nccl()
    ctx.close()
