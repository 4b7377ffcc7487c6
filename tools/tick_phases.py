"""Phase stamps of the fused tick (EWSJF_PHASES=1): per-CTA %globaltimer stamps of one
C3 tick, printed as median / max µs from the earliest CTA start.  Diagnostic only
(the stamps add a few global stores); run on a GPU box:

    EWSJF_PHASES=1 python tools/tick_phases.py [--partition rp|quantile] [--k 64]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_21758_b200 as E  # noqa: E402
import workload  # noqa: E402

SLOTS = {"start": 0, "issued": 10, "zero": 12, "setup": 1, "sample_landed": 15, "sample_tile": 26, "sample": 2, "pub": 13,
         "bound": 14, "thr": 3, "stream": 4, "rows_cut": 28, "counts": 29, "agg": 30, "pre_barrier": 5,
         "barrier": 6, "merge_rows": 20, "merge_filtered": 16, "merge_selected": 18, "merge_out": 19, "merge_rep0_end": 27, "merge": 7}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--partition", default="rp", choices=["rp", "quantile"])
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    assert os.environ.get("EWSJF_PHASES"), "set EWSJF_PHASES=1"
    dev = torch.device("cuda", 0)
    ctx = E.Context(0, max_pool=a.n, max_history=1_000_000, max_k=max(a.k, 64))
    hist = workload.heavy(1_000_000, 301)
    if a.partition == "rp":
        part, _, _ = E.partition(ctx, torch.from_numpy(hist).to(dev))
    else:
        part = E.make_partition(workload.quantile_bounds(hist, 32))
    pool = workload.pool("heavy", a.n, 302)
    t = [torch.from_numpy(pool[k]).to(dev) for k in ("len", "arrival", "cost")]
    q = torch.empty(a.n, dtype=torch.int32, device=dev)
    theta = E.meta(**workload.THETA0)
    sp = E.select_params(k=a.k, mode=0, now=workload.NOW)
    out = E.Outputs.alloc(a.k, dev)
    rows = []
    for i in range(5):
        E.tick(ctx, *t, part, theta, sp, qid_out=q, out=out, sync=False)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    for i in range(50):      # back to back: the event time of a launch in a stream of ticks
        E.tick(ctx, *t, part, theta, sp, qid_out=q, out=out, sync=False)
    torch.cuda.synchronize()
    tm = ctx.timing()
    ev_us = 1e3 * tm["tick_ms"] / max(tm["tick_launches"], 1)
    ctx.set_timing(False)
    for i in range(a.reps):
        E.tick(ctx, *t, part, theta, sp, qid_out=q, out=out, sync=False)
        torch.cuda.synchronize()
        ph = ctx.phases().astype(np.int64)
        st = ph[:, 0]
        t0 = st[st > 0].min()
        r = {}
        for name, s in SLOTS.items():
            v = ph[:, s]
            v = v[(v > 0) & (v >= t0) & (v < t0 + 10_000_000)]
            if len(v):
                r[name] = ((np.median(v) - t0) / 1e3, (v.max() - t0) / 1e3)
        pn = ph[:, 17]
        r["merge_pn_max"] = (float(pn[pn < 1_000_000].max()) if (pn < 1_000_000).any() else 0.0, 0.0)
        rows.append(r)
    res = {"n": a.n, "partition": a.partition, "k": a.k, "tick_us_event": ev_us,
           "ph": {name: "%.1f/%.1f" % tuple(np.median([r[name][j] for r in rows[2:] if name in r]) for j in (0, 1))
                  for name in list(SLOTS) + ["merge_pn_max"] if any(name in r for r in rows[2:])}}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
