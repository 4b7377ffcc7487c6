"""Driver for compute-sanitizer (memcheck / racecheck / synccheck): every kernel of
libewsjf once on small inputs -- the fused tick (SCORE and FIFO, gap requests and
bubbles included), the general tick path (> 64 queues), route, score_select,
the sharded local + merge, Refine-and-Prune (both prune variants reached at this
size: shared-memory tree) and the k-means-only partition, the Θ sweep, the
batch builder and online adjust.  Run as
    compute-sanitizer --tool memcheck python tests/sanitize_run.py
(profiles/*_sanitizer_*.log hold the committed results)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_21758_b200 as E  # noqa: E402
import workload  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    n = 20_000
    ctx = E.Context(0, max_pool=n, max_history=50_000, max_k=64, max_sweep=n)
    hist = torch.from_numpy(workload.heavy(50_000, 1)).to(dev)
    part, _, _ = E.partition(ctx, hist)
    part_km, _, _ = E.partition(ctx, hist, E.partition_params(kmeans_k=10))
    E.online_adjust(ctx, torch.from_numpy(workload.heavy(20_000, 2)).to(dev), type(part).from_buffer_copy(part))
    pool = workload.pool("heavy", n, 3)
    ln, ar, co = (torch.from_numpy(pool[k]).to(dev) for k in ("len", "arrival", "cost"))
    q = torch.empty_like(ln)
    th = E.meta(**workload.THETA0)
    for mode in (0, 1):
        E.tick(ctx, ln, ar, co, part, th, E.select_params(k=16, mode=mode), qid_out=q)
        E.tick(ctx, ln, ar, None, part_km, th, E.select_params(k=16, mode=mode), qid_out=q)
    holes = E.make_partition([(32, 100), (100, 2001), (2001, 5000), (7000, 40000)])
    E.tick(ctx, ln, ar, co, holes, th, E.select_params(k=16, mode=0), qid_out=q)        # Alg. 2 + bubbles
    many = E.make_partition([(1 + 40 * i, 41 + 40 * i) for i in range(100)] + [(4001, 40000)])
    E.tick(ctx, ln, ar, co, many, th, E.select_params(k=8, mode=0), qid_out=q)         # > 64 queues: general path
    qid, _ = E.route(ctx, ln, part)
    E.score_select(ctx, ln, ar, co, qid, part, E.weights_from_meta(th, part), E.select_params(k=16))
    out = E.tick(ctx, ln, ar, co, part, th, E.select_params(k=64, mode=1), qid_out=q)
    E.batch_build(ctx, ln, out, out.summary["n_queues"], 64, 20_000)
    thetas = [E.meta(**t) for t in workload.random_thetas(8, 4)]
    E.score_select_sweep(ctx, ln, ar, co, qid, part, thetas, E.select_params(k=8))
    ln_hot = ln.clone()
    ln_hot[:3000] = 100                  # one length with > 1024 records: the sweep's CTA-per-length path
    qid_hot, _ = E.route(ctx, ln_hot, part)
    E.score_select_sweep(ctx, ln_hot, ar, co, qid_hot, part, thetas, E.select_params(k=8))
    # A1 long tail: lengths >= 2^20 through the overflow list
    h_long = workload.heavy(50_000, 5)
    h_long[:300] = np.random.default_rng(6).integers(1 << 20, 1 << 24, size=300)
    E.partition(ctx, torch.from_numpy(h_long).to(dev))
    recs = [E.tick_local(ctx, ln[a:b], ar[a:b], co[a:b], a, part, th, E.select_params(k=16), qid_out=q[a:b]).clone()
            for a, b in (workload.shard_range(n, r, 2) for r in range(2))]
    E.tick_merge(ctx, torch.cat(recs), 2, 0, n // 2, q[: n // 2], E.make_partition(
        [(x["min_len"], x["max_len"]) for x in part.queues()]), th, E.select_params(k=16))
    torch.cuda.synchronize()
    ctx.close()
    if os.environ.get("SANITIZE_BIG"):   # the pipelined ewsjf_tick_host (pools >= 2M)
        nb = 2_100_000
        big = E.Context(0, max_pool=nb, max_history=0, max_k=16)
        pb = workload.pool("heavy", nb, 7)
        hl, ha, hc = (torch.from_numpy(pb[k]).pin_memory() for k in ("len", "arrival", "cost"))
        E.tick_host(big, hl, ha, hc, part, th, E.select_params(k=16), qid_out=torch.empty(nb, dtype=torch.int32).pin_memory())
        torch.cuda.synchronize()
        big.close()
    print("sanitize driver done")


if __name__ == "__main__":
    main()
