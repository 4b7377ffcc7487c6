"""SURVEY §8b boundary contract: the ctx owns all scratch, allocated once, so no
hot call (tick, score_select, route, Θ sweep, batch build, sharded tick) makes
a cudaMalloc / cudaMallocHost / cudaFree.  The library counts every allocation
and free it makes (ewsjf_alloc_count); the count must not move across hot calls."""
import numpy as np
import pytest
import torch

import workload

pytestmark = pytest.mark.gpu


def test_hot_calls_do_not_allocate():
    import paper_2601_21758_b200 as E
    dev = torch.device("cuda", 0)
    n = 300_000
    ctx = E.Context(0, max_pool=n, max_history=100_000, max_k=256, max_sweep=n)
    part, _, _ = E.partition(ctx, torch.from_numpy(workload.heavy(100_000, 3)).to(dev))
    pool = workload.pool("heavy", n, 4)
    ln, ar, co = (torch.from_numpy(pool[k]).to(dev) for k in ("len", "arrival", "cost"))
    q = torch.empty_like(ln)
    th = E.meta(**workload.THETA0)
    outs = {k: E.Outputs.alloc(k, dev) for k in (64, 256)}
    thetas = [E.meta(**t) for t in workload.random_thetas(20, 5)]
    sw_outs = [E.Outputs.alloc(16, dev) for _ in thetas]
    ids = torch.empty(256, dtype=torch.int64, device=dev)
    info = torch.empty(4, dtype=torch.int64, device=dev)
    w = E.weights_from_meta(th, part)

    def hot():
        E.tick(ctx, ln, ar, co, part, th, E.select_params(k=64, mode=0), qid_out=q, out=outs[64], sync=False)
        E.tick(ctx, ln, ar, co, part, th, E.select_params(k=256, mode=1), qid_out=q, out=outs[256], sync=False)
        E.batch_build(ctx, ln, outs[256], part.n, 256, 65536, ids_out=ids, info_out=info)
        E.score_select(ctx, ln, ar, co, q, part, w, E.select_params(k=64, mode=0), out=outs[64], sync=False)
        E.score_select_sweep(ctx, ln, ar, co, q, part, thetas, E.select_params(k=16, mode=0), outs=sw_outs)
        E.route(ctx, ln, part, qid_out=q)
        torch.cuda.synchronize()

    hot()                                   # first calls: LUT upload etc. (no allocation either)
    before = E.alloc_count()
    for _ in range(3):
        hot()
    assert E.alloc_count() == before, (before, E.alloc_count())
    ctx.close()
