import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle as O, workload
import paper_2601_21758_b200 as E
from tests.parity import compare_selection, gpu_result, to_gpu_partition
s, opart, _ = O.partition(workload.bimodal(10_000, 101))
ctx = E.Context(0, max_pool=1<<22, max_history=1<<20, max_k=64)
print("ctas", ctx.num_ctas)
for n in (1000, 700_001):
  pool = workload.pool("bimodal", n, 102)
  for mode in (0,1):
    qid = torch.empty(n, dtype=torch.int32, device="cuda")
    out = E.tick(ctx, torch.from_numpy(pool["len"]).cuda(), torch.from_numpy(pool["arrival"]).cuda(), torch.from_numpy(pool["cost"]).cuda(), to_gpu_partition(E, opart), E.meta(**workload.THETA0), E.select_params(k=64, mode=mode), qid_out=qid)
    torch.cuda.synchronize()
    print("summary", out.summary)
    ref = O.tick(pool["len"], pool["arrival"], pool["cost"], opart, O.meta(**workload.THETA0), O.select_params(k=64, mode=mode))
    phi, _ = O.score_all(pool["len"], pool["arrival"], pool["cost"], ref["qid"], ref["partition"], O.meta(**workload.THETA0), O.select_params(k=64, mode=mode))
    print("qid eq", (qid.cpu().numpy() == ref["qid"]).all())
    g = gpu_result(out)
    print("count", g["count"][:5], ref["count"][:5])
    print("head", g["head_id"][:5], ref["head_id"][:5])
    print("top", g["topk_id"][31][:8], ref["topk_id"][31][:8])
    try:
        rep = compare_selection(g, ref, phi, pool["arrival"], mode, 64)
        print("PARITY OK", n, mode, rep.near_ties)
    except AssertionError as e:
        print("PARITY FAIL", n, mode, e)
