"""Run the C3 fused tick a few times (for ncu captures): python tools/tick_loop.py [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_21758_b200 as E  # noqa: E402
import workload  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
part_kind = sys.argv[2] if len(sys.argv) > 2 else "rp"
dev = torch.device("cuda", 0)
n = 10_000_000
ctx = E.Context(0, max_pool=n, max_history=1_000_000, max_k=64)
hist = workload.heavy(1_000_000, 301)
if part_kind == "rp":
    part, _, _ = E.partition(ctx, torch.from_numpy(hist).to(dev))
else:
    part = E.make_partition(workload.quantile_bounds(hist, 32))
pool = workload.pool("heavy", n, 302)
t = [torch.from_numpy(pool[k]).to(dev) for k in ("len", "arrival", "cost")]
q = torch.empty(n, dtype=torch.int32, device=dev)
out = E.Outputs.alloc(64, dev)
theta = E.meta(**workload.THETA0)
sp = E.select_params(k=64, mode=0, now=workload.NOW)
for i in range(reps):
    E.tick(ctx, *t, part, theta, sp, qid_out=q, out=out, sync=False)
torch.cuda.synchronize()
print("ok")
