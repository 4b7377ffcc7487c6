#!/usr/bin/env python
"""Benchmark of the EWSJF scheduling tick on B200 (BASELINE.json metric).

Workload (N=1, config C3 = BASELINE.json configs[2], the config the metric is
quoted on): 10,000,000 pending requests with heavy-tailed prompt lengths per
GPU, SoA (len int32, arrival fp32, cost fp32) resident in HBM; the policy is the
Refine-and-Prune partition of a 1M heavy-tailed history computed on the GPU by
ewsjf_partition (strategic loop, published before the timed region; its own
time is reported under "strategic").  One step = one ewsjf_tick: route (A8) +
bubbles (A9) + weights (A7) + Eq. 4 score (A10) + per-queue top-64 / head /
ArgMax (A11).  Multi-GPU: weak scaling, every rank owns 10M requests (global
ids rank*10M + i), candidates all-gathered over NCCL (tick_sharded).

L2: 3 rotating pool copies (3 x 160 MB > 126 MB L2), so no step reads inputs
left in L2 by the previous step.

``--impl reference`` times the CPU oracle (the reference arm of this tier) on
the same workload, a bounded sample per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workload  # noqa: E402

METRIC = "requests scored+routed+selected/s per tick at 10M pending; % HBM roofline"
UNIT = "req/s"
BYTES_PER_REQ = 16          # len 4 + arrival 4 + cost 4 read, qid 4 written


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=10_000_000, help="pending requests per GPU")
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--mode", default="score", choices=["score", "fifo"])
    ap.add_argument("--partition", default="rp", choices=["rp", "quantile"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the C5 Θ-sweep measurement")
    ap.add_argument("--sweep-thetas", type=int, default=256)
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 100M-history Refine-and-Prune measurement")
    ap.add_argument("--no-traffic", action="store_true", help="skip the in-run ncu dram-bytes probe")
    ap.add_argument("--no-extra", action="store_true", help="skip the C1/C2/balanced-C3 lines")
    ap.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: --n is the TOTAL pool, split by index across the ranks")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 8]
        busy = [r for r in rows if r[2].isdigit() and int(r[2]) > 0] or rows
        sm = [float(r[0]) for r in busy if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in busy for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "samples_busy": len(busy)}


def oracle_rate(pool, opart, K, mode, sample_n, repeats=1):
    """The CPU oracle (test infrastructure) on a bounded sample of the workload."""
    import oracle as O
    sp = O.select_params(k=K, mode=mode, now=workload.NOW)
    th = O.meta(**workload.THETA0)
    ln, ar, co = pool["len"][:sample_n], pool["arrival"][:sample_n], pool["cost"][:sample_n]
    ts = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        O.tick(ln, ar, co, opart, th, sp)
        ts.append(time.perf_counter() - t0)
    return sample_n / statistics.median(ts), statistics.median(ts)


def oracle_partition(hist):
    import oracle as O
    s, part, _ = O.partition(hist)
    return part


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    """Reference arm of this tier: the CPU oracle, as it stands, on the box's host cores."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    mode = 0 if args.mode == "score" else 1
    hist = workload.heavy(1_000_000, 301)
    opart = oracle_partition(hist)
    pool = workload.pool("heavy", args.n, 302)
    # size each step's sample so the whole warmup+steps run takes ~1-2 minutes
    _, t_cal = oracle_rate(pool, opart, args.k, mode, 200_000)
    per_req = t_cal / 200_000
    budget = 90.0
    sample_n = int(max(2_000, min(args.n, budget / max(args.steps + args.warmup, 1) / per_req)))
    for _ in range(args.warmup):
        oracle_rate(pool, opart, args.k, mode, sample_n)
    ts = []
    for _ in range(args.steps):
        _, t = oracle_rate(pool, opart, args.k, mode, sample_n)
        ts.append(t)
    tot = sum(ts)
    value = sample_n * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, opart_source="oracle Refine-and-Prune of heavy(1M, seed 301)"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"first {sample_n} requests of the C3 pool per step (oracle tick: route, "
                                   f"bubbles, weights, Eq. 4 score, per-queue full sort), single thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_sweep(E, ctx, dev, args, rank=0, ws=1, group=None):
    """C5 (BASELINE configs[4]): 256 Θ x 1M snapshot, K=16, SCORE mode; at N GPUs the
    Θ are split by rank (32 per GPU at 8) and each rank sweeps its share
    over the same (replicated) snapshot, no exchange; time = max over ranks.
    ALU-bound: each (request, Θ) pair is 3 fp32 FMA-pipe ops (FMUL + 2 FFMA) and one
    FSETP on the hot path, so the peak is 148 SMs x 128 fp32 lanes x clock / 4."""
    import torch
    n = 1_000_000
    hist = torch.from_numpy(workload.bimodal(1_000_000, 201)).to(dev)
    c2part, _, _ = E.partition(ctx, hist)
    pool = workload.pool("bimodal", n, 501)
    ln, ar, co = (torch.from_numpy(pool[k]).to(dev) for k in ("len", "arrival", "cost"))
    qid, rsum = E.route(ctx, ln, c2part)
    all_t = workload.random_thetas(args.sweep_thetas, 502)
    lo_t, hi_t = workload.shard_range(len(all_t), rank, ws)
    thetas = E.meta_array([E.meta(**t) for t in all_t[lo_t:hi_t]])
    sp = E.select_params(k=16, mode=0, now=workload.NOW)
    sctx = E.Context(dev.index or 0, max_pool=n, max_history=0, max_k=64, max_sweep=n)
    outs = E.score_select_sweep(sctx, ln, ar, co, qid, c2part, thetas, sp)
    for _ in range(2):
        E.score_select_sweep(sctx, ln, ar, co, qid, c2part, thetas, sp, outs=outs)
    torch.cuda.synchronize()
    reps = 10
    sctx.set_timing(True)
    l0 = sctx.timing()["launches"]
    if group is not None:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        E.score_select_sweep(sctx, ln, ar, co, qid, c2part, thetas, sp, outs=outs)
    e1.record()
    torch.cuda.synchronize()
    tm = sctx.timing()
    ms = e0.elapsed_time(e1) / reps
    if group is not None:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    pairs = n * len(all_t)                      # all ranks together
    ffma = sctx.ffma_rate()            # measured fp32 FFMA/s on this box
    peak = ffma / 4 * ws               # 4 fp32-pipe instructions per (request, Θ) pair, all ranks
    achieved = pairs / (ms / 1e3)
    sctx.close()
    return {"workload": "C5: 256 Θ uniform in S:500 bounds (seed 502) x 1M bimodal snapshot (seed 501) routed by "
                        "the GPU Refine-and-Prune partition of bimodal(1M, seed 201); K=16, SCORE",
            "metric": "(request, Θ) pairs scored+selected/s", "value": achieved, "ms_per_sweep": ms,
            "thetas": len(all_t), "thetas_per_rank": len(thetas), "ranks": ws, "snapshot": n, "queues": c2part.n,
            "kernel_ms_per_sweep": tm["sweep_ms"] / reps, "launches_per_sweep": (tm["launches"] - l0) / reps,
            "graph_launches_per_sweep": tm["sweep_launches"] / reps,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "pairs/s",
                         "frac": achieved / peak,
                         "peak_source": "measured: ewsjf_diag_ffma_rate (FFMA throughput microbenchmark) / "
                                        "4 fp32-pipe instructions per pair", "ffma_per_s": ffma},
            "candidates_inserted_last_sweep": tm["candidates_inserted"],
            "records_after_prefilter": tm["sweep_records"]}


def run_batch(E, ctx, part, theta, copies, dev, n, max_req=256, max_tok=65536, reps=20):
    """Alg. 1's Batch Builder after a FIFO-mode tick at the C3 size
    (k = max_requests so every queue's pullable FIFO prefix is in its row)."""
    import torch
    sp = E.select_params(k=max_req, mode=1, now=workload.NOW)
    out = E.Outputs.alloc(max_req, dev)
    ids = torch.empty(max_req, dtype=torch.int64, device=dev)
    info = torch.empty(4, dtype=torch.int64, device=dev)
    ln, ar, co, q = copies[0]
    s = E.tick(ctx, ln, ar, co, part, theta, sp, qid_out=q, out=out)
    nq = s.summary["n_queues"]
    for _ in range(3):
        E.batch_build(ctx, ln, out, nq, max_req, max_tok, ids_out=ids, info_out=info)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    for i in range(reps):
        l2, a2, c2, q2 = copies[i % 3]
        E.tick(ctx, l2, a2, c2, part, theta, sp, qid_out=q2, out=out, sync=False)
        E.batch_build(ctx, l2, out, nq, max_req, max_tok, ids_out=ids, info_out=info)
    torch.cuda.synchronize()
    tm = ctx.timing()
    inf = info.cpu().tolist()
    return {"workload": f"FIFO tick (k={max_req}) over the C3 pool + Alg. 1 batch build "
                        f"(max_requests={max_req}, max_tokens={max_tok})",
            "batch_kernel_us": 1e3 * tm["batch_ms"] / max(tm["batch_launches"], 1),
            "fifo_tick_kernel_ms": tm["tick_ms"] / max(tm["tick_launches"], 1),
            "fifo_merge_kernel_ms": tm["merge_ms"] / max(tm["merge_launches"], 1),
            "batch_size": inf[0], "batch_tokens": inf[1], "status": inf[2], "primary": inf[3]}


def run_c4(E, dev, local, kind="heavy", seed=402, reps=3):
    """C4 (BASELINE configs[3]): Refine-and-Prune over a 100M history on one GPU
    (SURVEY §8d seeds: bimodal 401, heavy 402)."""
    import torch
    hist = torch.from_numpy(workload.lengths(kind, 100_000_000, seed)).to(dev)
    cctx = E.Context(local, max_pool=1024, max_history=100_000_000, max_k=8)
    E.partition(cctx, hist)
    cctx.set_timing(True)
    sts = []
    for _ in range(reps):
        part, st, _ = E.partition(cctx, hist)
        sts.append(st)
    tm = cctx.timing()
    cctx.close()
    med = sorted(sts, key=lambda x: x["ms_total"])[len(sts) // 2]
    peak, src = peaks()
    hist_gbs = 4e8 / (med["ms_hist"] / 1e3) / 1e9
    return {"workload": f"C4: Refine-and-Prune of {kind}(100M, seed {seed}), alpha=2, max_queues=32, MIN_U",
            "ms": med["ms_total"], "stages_ms": {k: med[k] for k in ("ms_hist", "ms_kmeans", "ms_refine", "ms_prune")},
            "kernel_ms_sum": tm["partition_ms"] / reps, "launches": tm["partition_launches"] / reps,
            "distinct": med["distinct"], "segments": med["segments"], "merges": med["merges"], "queues": part.n,
            "hist_roofline": {"bound": "hbm", "achieved": hist_gbs, "peak": peak, "unit": "GB/s",
                              "frac": hist_gbs / peak, "bytes": 4e8, "peak_source": src}}


def median_ms(fn, reps=5, warm=1):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return statistics.median(ts)


def tick_kernel_us(E, ctx, pool_t, part, theta, sp, reps=50):
    """Median-free mean of the tick kernel time (CUDA events on the ctx stream) over reps launches."""
    import torch
    ln, ar, co, q = pool_t
    out = E.Outputs.alloc(sp.k, ln.device)
    for _ in range(5):
        E.tick(ctx, ln, ar, co, part, theta, sp, qid_out=q, out=out, sync=False)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        E.tick(ctx, ln, ar, co, part, theta, sp, qid_out=q, out=out, sync=False)
    e1.record()
    torch.cuda.synchronize()
    tm = ctx.timing()
    ctx.set_timing(False)
    return {"kernel_us": 1e3 * tm["tick_ms"] / max(tm["tick_launches"], 1), "step_us": 1e3 * e0.elapsed_time(e1) / reps}


def oracle_rp_ms(hist, **kw):
    import oracle as O
    t0 = time.perf_counter()
    s, part, st = O.partition(hist, **kw)
    return 1e3 * (time.perf_counter() - t0), part


def run_extra(E, dev, local, args, peak):
    """SURVEY §8d rows besides the headline: C1 (1k pending, 10k history, one tick:
    latency), C2 (100k pending, 1M bimodal history: R&P + tick) and the C3 tick on the
    balanced 32-quantile partition (SURVEY hard part 4).  The oracle beside each R&P."""
    import torch
    res = {}
    theta = E.meta(**workload.THETA0)
    sp = E.select_params(k=64, mode=0, now=workload.NOW)
    for name, hseed, pseed, npool, nhist in (("c1", 101, 102, 1_000, 10_000), ("c2", 201, 202, 100_000, 1_000_000)):
        ctx = E.Context(local, max_pool=npool, max_history=nhist, max_k=64)
        hist = workload.bimodal(nhist, hseed)
        hd = torch.from_numpy(hist).to(dev)
        rp_ms = median_ms(lambda: E.partition(ctx, hd), reps=5)
        part, pst, _ = E.partition(ctx, hd)
        pool = workload.pool("bimodal", npool, pseed)
        pt = tuple(torch.from_numpy(pool[k]).to(dev) for k in ("len", "arrival", "cost")) + \
            (torch.empty(npool, dtype=torch.int32, device=dev),)
        tk = tick_kernel_us(E, ctx, pt, part, theta, sp)
        o_ms, _ = oracle_rp_ms(hist)
        res[name] = {"workload": f"{name.upper()}: history bimodal({nhist}, seed {hseed}), pool bimodal({npool}, "
                                 f"seed {pseed}); GPU R&P + fused tick (K=64, SCORE)",
                     "refine_and_prune_ms_median5": rp_ms,
                     "stages_ms": {k: pst[k] for k in ("ms_hist", "ms_kmeans", "ms_refine", "ms_prune")},
                     "segments": pst["segments"], "merges": pst["merges"], "queues": part.n,
                     "tick_kernel_us": tk["kernel_us"], "tick_step_us": tk["step_us"],
                     "tick_req_per_s": npool / (tk["step_us"] * 1e-6),
                     "one_tick_total_us": 1e3 * rp_ms + tk["step_us"],
                     "oracle_refine_and_prune_ms": o_ms}
        ctx.close()
    # C3 on the balanced 32-quantile partition of the same history
    n = args.n
    ctx = E.Context(local, max_pool=n, max_history=0, max_k=64)
    qpart = E.make_partition(workload.quantile_bounds(workload.heavy(1_000_000, 301), 32))
    pool = workload.pool("heavy", n, 302)
    pt = tuple(torch.from_numpy(pool[k]).to(dev) for k in ("len", "arrival", "cost")) + \
        (torch.empty(n, dtype=torch.int32, device=dev),)
    tk = tick_kernel_us(E, ctx, pt, qpart, theta, sp, reps=100)
    gbs = BYTES_PER_REQ * n / (tk["kernel_us"] * 1e-6) / 1e9
    res["c3_balanced"] = {"workload": "C3 pool, balanced 32-quantile partition of heavy(1M, seed 301), K=64, SCORE",
                          "tick_kernel_us": tk["kernel_us"], "tick_step_us": tk["step_us"],
                          "req_per_s": n / (tk["step_us"] * 1e-6),
                          "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                                       "frac": gbs / peak}}
    ctx.close()
    return res


def measure_traffic(n, timeout=300):
    """dram__bytes_read.sum + dram__bytes_write.sum of the fused tick kernel, measured
    in this run by re-executing this script's --traffic-probe mode under ncu (one GPU,
    one profiled launch after warm-up).  Returns (bytes per launch, note)."""
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none",
           "-k", "regex:ftick_kernel", "-s", "3", "-c", "1", "--csv", sys.executable, os.path.abspath(__file__),
           "--traffic-probe", "--n", str(n)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    except Exception as e:  # noqa: BLE001
        return None, f"ncu probe failed: {e}"
    tot = 0.0
    seen = 0
    for line in r.stdout.splitlines():
        if "dram__bytes_read.sum" in line or "dram__bytes_write.sum" in line:
            f = [x.strip('"') for x in line.split('","')]
            try:
                unit, val = f[-2], float(f[-1].strip('"').replace(",", ""))
            except Exception:  # noqa: BLE001
                continue
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
            tot += val * scale
            seen += 1
    if seen < 2:
        return None, "ncu output not parsed: " + (r.stdout[-300:] + r.stderr[-300:]).replace("\n", " ")
    return tot, "ncu dram__bytes_read.sum + dram__bytes_write.sum, one launch of ewsjf::ftick_kernel, this run"


def traffic_probe(args):
    import torch
    import paper_2601_21758_b200 as E
    dev = torch.device("cuda", 0)
    ctx = E.Context(0, max_pool=args.n, max_history=1_000_000, max_k=64)
    part, _, _ = E.partition(ctx, torch.from_numpy(workload.heavy(1_000_000, 301)).to(dev))
    pool = workload.pool("heavy", args.n, 302)
    ln, ar, co = (torch.from_numpy(pool[k]).to(dev) for k in ("len", "arrival", "cost"))
    q = torch.empty_like(ln)
    out = E.Outputs.alloc(args.k, dev)
    for _ in range(5):
        E.tick(ctx, ln, ar, co, part, E.meta(**workload.THETA0), E.select_params(k=args.k, mode=0), qid_out=q,
               out=out, sync=False)
    torch.cuda.synchronize()


_SHARD = {}


def _oracle_shard(a):
    import oracle as O
    lo, hi, k, mode = a
    pool, opart = _SHARD["pool"], _SHARD["part"]
    sp = O.select_params(k=k, mode=mode, now=workload.NOW)
    t0 = time.perf_counter()
    O.tick(pool["len"][lo:hi], pool["arrival"][lo:hi], pool["cost"][lo:hi], opart, O.meta(**workload.THETA0), sp,
           global_base=lo)
    return hi - lo, time.perf_counter() - t0


def oracle_all_cores(pool, opart, n_sample, k, mode):
    """The oracle on every host core: the first n_sample requests of the C3 pool split
    by index into one shard per core (the natural parallel form of O8-O10's
    per-request map; each shard a full oracle tick with global ids), wall time of
    the whole parallel map."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    _SHARD["pool"] = {k: pool[k][:n_sample] for k in ("len", "arrival", "cost")}
    _SHARD["part"] = opart
    bounds = [(i * n_sample // cores, (i + 1) * n_sample // cores) for i in range(cores)]
    ctxm = mp.get_context("fork")
    with ctxm.Pool(cores) as pp:
        pp.map(_oracle_shard, [(0, 1000, k, mode)] * cores)   # warm (page-in)
        t0 = time.perf_counter()
        r = pp.map(_oracle_shard, [(lo, hi, k, mode) for lo, hi in bounds])
        wall = time.perf_counter() - t0
    return sum(x for x, _ in r) / wall, wall, cores


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    return None


def config_dict(args, opart_source):
    return {"workload": "C3: 10M pending requests per GPU, heavy-tailed lengths (80% lognormal(ln128,0.6) "
                        "32..2047, 20% Pareto(1.5) 2048..32768), route + score + per-queue top-k",
            "pending_per_gpu": args.n, "k": args.k, "mode": args.mode, "partition": opart_source,
            "theta": workload.THETA0, "now_s": workload.NOW, "cost_field": True,
            "l2": "3 rotating pool copies (3 x 160 MB > 126 MB L2)",
            "parallelism": f"index-sharded x{args.gpus}, NCCL all-gather of candidates" if args.gpus > 1 else "1 GPU"}


def main():
    args = parse()
    if args.traffic_probe:
        traffic_probe(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import paper_2601_21758_b200 as E
    from paper_2601_21758_b200 import _lib as L

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    mode = L.SELECT_SCORE if args.mode == "score" else L.SELECT_FIFO
    if args.strong:       # the TOTAL pool split by index (rank r owns [floor(rN/P), floor((r+1)N/P)))
        lo_r, hi_r = workload.shard_range(args.n, rank, ws)
        n = hi_r - lo_r
    else:
        lo_r, n = rank * args.n, args.n
    ctx = E.Context(local, max_pool=n, max_history=1_000_000, max_k=max(args.k, 64))

    # ---- strategic loop: Refine-and-Prune on the GPU (published before the timed region)
    hist = torch.from_numpy(workload.heavy(1_000_000, 301)).to(dev)
    strategic = {}
    if args.partition == "rp":
        part, pst, _ = E.partition(ctx, hist)           # cold (first call)
        cold_ms = pst["ms_total"]
        sts = []
        for _ in range(5):                              # warm: median of 5
            _, st_, _ = E.partition(ctx, hist)
            sts.append(st_)
        pst = sorted(sts, key=lambda x: x["ms_total"])[2]
        strategic = {"refine_and_prune_ms": pst["ms_total"], "refine_and_prune_ms_cold": cold_ms,
                     "timing": "median of 5 warm calls (CUDA events per stage)", "history": 1_000_000,
                     "queues": part.n,
                     "stages_ms": {k: pst[k] for k in ("ms_hist", "ms_kmeans", "ms_refine", "ms_prune")},
                     "distinct": pst["distinct"], "segments": pst["segments"], "merges": pst["merges"]}
        if rank == 0 and not args.no_cpu_baseline:
            o_ms, _ = oracle_rp_ms(workload.heavy(1_000_000, 301))
            strategic["oracle_refine_and_prune_ms"] = o_ms
        psrc = "GPU Refine-and-Prune (ewsjf_partition) of heavy(1M, seed 301), alpha=2, max_queues=32, MIN_U"
    else:
        part = E.make_partition(workload.quantile_bounds(workload.heavy(1_000_000, 301), 32))
        psrc = "balanced 32-quantile partition of heavy(1M, seed 301)"
    theta = E.meta(**workload.THETA0)
    sp = E.select_params(k=args.k, mode=mode, now=workload.NOW)
    if args.partition == "rp":
        # online adjust mode (R31) of that partition from a 1M recent window (on a copy)
        win = torch.from_numpy(workload.heavy(1_000_000, 303)).to(dev)
        padj = type(part).from_buffer_copy(part)
        E.online_adjust(ctx, win, padj)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            padj = type(part).from_buffer_copy(part)
            moved = E.online_adjust(ctx, win, padj)
        strategic["online_adjust"] = {"window": 1_000_000, "ms_per_call": (time.perf_counter() - t0) * 1e3 / 5,
                                      "boundaries_moved": moved, "max_shift": 0.25,
                                      "note": "synchronous call incl. window histogram + one CTA per boundary"}

    # ---- pool: this rank's 10M shard, 3 rotating copies in HBM
    if args.strong:
        full = workload.pool("heavy", args.n, 302)
        pool = {k: v[lo_r:hi_r].copy() for k, v in full.items()}
        del full
    else:
        pool = workload.pool("heavy", n, 302 + 1000 * rank)
    copies = []
    for c in range(3):
        copies.append((torch.from_numpy(pool["len"]).to(dev), torch.from_numpy(pool["arrival"]).to(dev),
                       torch.from_numpy(pool["cost"]).to(dev), torch.empty(n, dtype=torch.int32, device=dev)))
    out = E.Outputs.alloc(args.k, dev)
    base = lo_r
    # N > 1: the library's own NCCL communicator (ewsjf_ctx_init_nccl; the unique id goes
    # over the torch process group once): ewsjf_tick then runs local -> ncclAllGather ->
    # merge on the ctx stream.  torch's all_gather (tick_sharded) only if that fails.
    lib_nccl = False
    if ws > 1:
        try:
            ctx.init_nccl(rank=rank, world=ws, group=group)
            lib_nccl = True
        except Exception as e:  # noqa: BLE001
            print(f"bench: library NCCL unavailable ({e}); torch all_gather instead", file=sys.stderr)

    def step(i):
        ln, ar, co, q = copies[i % 3]
        if ws > 1 and not lib_nccl:
            E.tick_sharded(ctx, ln, ar, co, base, part, theta, sp, group=group, qid_out=q, out=out, sync=False)
        else:
            E.tick(ctx, ln, ar, co, part, theta, sp, global_base=base, qid_out=q, out=out, sync=False)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    summary = E.tick(ctx, *copies[0][:3], part, theta, sp, global_base=base, qid_out=copies[0][3]).summary \
        if ws == 1 else None

    sampler = ClockSampler(local)
    sampler.start()
    t_wait = time.time()
    while not sampler.rows and time.time() - t_wait < 5.0:   # nvidia-smi is sampling before the timed region
        time.sleep(0.02)
    # timed region: K steps between a barrier + synchronize on both sides
    if group is not None:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ctx.set_timing(True)
    launches0 = ctx.timing()["launches"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        step(i)
    e1.record()
    torch.cuda.synchronize()
    if group is not None:
        torch.distributed.barrier()
    ms = e0.elapsed_time(e1)
    tm = ctx.timing()
    clocks = sampler.stop()
    if group is not None:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = (args.n if args.strong else n * ws) / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel (the partial tick pass)
    peak, peak_src = peaks()
    tick_ms = tm["tick_ms"] / max(tm["tick_launches"], 1)
    merge_ms = tm["merge_ms"] / max(tm["merge_launches"], 1)
    achieved = BYTES_PER_REQ * n / (tick_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None, "kernel": "ewsjf::ftick_kernel (fused: streaming route+score+filter, sample bound, grid barrier, per-queue merge)",
                "algorithmic_bytes_per_launch": BYTES_PER_REQ * n, "kernel_ms": tick_ms,
                "merge_kernel_ms": merge_ms, "peak_source": peak_src,
                "share_of_step": tick_ms / ms_per_step if ms_per_step else None}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None,
        "dtype": "f32", "data": "synthetic", "config": config_dict(args, psrc), "roofline": roofline,
        "gpu_launches": int(tm["launches"] - launches0), "clocks": clocks, "strategic": strategic,
        "tick_summary": summary,
    }
    if ws > 1:
        line["exchange"] = ("library NCCL all-gather inside ewsjf_tick (ewsjf_ctx_init_nccl)" if lib_nccl
                            else "torch.distributed all_gather_into_tensor between ewsjf_tick_local / ewsjf_tick_merge")

    # ---- e2e through the C ABI with host buffers (H2D + D2H inside the timed region)
    if not args.no_e2e and ws == 1:
        hl = torch.from_numpy(pool["len"]).pin_memory()
        ha = torch.from_numpy(pool["arrival"]).pin_memory()
        hc = torch.from_numpy(pool["cost"]).pin_memory()
        hq = torch.empty(n, dtype=torch.int32).pin_memory()
        res = None
        for _ in range(2):
            res = E.tick_host(ctx, hl, ha, hc, part, theta, sp, qid_out=hq, results=res)
        k_e2e = max(3, min(20, args.steps // 20))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            res = E.tick_host(ctx, hl, ha, hc, part, theta, sp, qid_out=hq, results=res)
        dt = (time.perf_counter() - t0) / k_e2e
        out_bytes = sum(v.numel() * v.element_size() for k, v in res.items() if k != "summary")
        line["e2e"] = {"value": n / dt, "unit": UNIT, "h2d_bytes_per_step": 12 * n,
                       "d2h_bytes_per_step": 4 * n + out_bytes, "ms_per_step": 1e3 * dt, "steps": k_e2e,
                       "path": "ewsjf_tick_host (pinned host SoA in, qid + results out)"}

    # ---- C5: the meta-optimizer's Θ sweep (A12) over a 1M bimodal snapshot routed by
    # the GPU Refine-and-Prune partition of bimodal(1M, seed 201) (C2's partition)
    if not args.no_sweep:
        line["sweep"] = run_sweep(E, ctx, dev, args, rank, ws, group)
    if ws == 1 and not args.no_c4:
        line["c4"] = run_c4(E, dev, local, "heavy", 402)
        line["c4_bimodal"] = run_c4(E, dev, local, "bimodal", 401)
    if ws == 1 and not args.no_extra:
        line.update(run_extra(E, dev, local, args, peak))
    if ws == 1 and args.k <= 256:
        bctx = E.Context(local, max_pool=n, max_history=0, max_k=256)
        line["batch"] = run_batch(E, bctx, part, theta, copies, dev, n)
        bctx.close()

    # ---- the oracle beside it (rank 0, N=1 only), bounded sample
    if not args.no_cpu_baseline and ws == 1 and rank == 0:
        opart = oracle_partition(workload.heavy(1_000_000, 301)) if args.partition == "rp" else None
        if opart is None:
            import oracle as O
            opart = O.make_partition(workload.quantile_bounds(workload.heavy(1_000_000, 301), 32))
        sample_n = 2_000_000
        omode = 0 if args.mode == "score" else 1
        rate, secs = oracle_rate(pool, opart, args.k, omode, sample_n)
        arate, asecs, cores = oracle_all_cores(pool, opart, 4_000_000, args.k, omode)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
                                "sample": f"first {sample_n} requests of the C3 pool, one oracle tick "
                                          f"({secs:.1f} s, single-threaded C fp64)",
                                "host_cores_available": os.cpu_count(), "cpu_model": cpu_model(),
                                "all_cores": {"value": arate, "unit": UNIT, "cores": cores,
                                              "sample": f"first 4,000,000 requests of the C3 pool split by index "
                                                        f"into {cores} shards, one oracle tick per shard in "
                                                        f"{cores} processes ({asecs:.1f} s wall)"}}
        # parity on that sample: GPU tick vs the oracle (ids exact up to near-ties)
        try:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            import oracle as O
            from parity import compare_selection, gpu_result, to_gpu_partition
            ln_s, ar_s, co_s = (torch.from_numpy(pool[k][:sample_n].copy()).to(dev) for k in ("len", "arrival", "cost"))
            qs = torch.empty_like(ln_s)
            pctx = E.Context(local, max_pool=sample_n, max_history=0, max_k=max(args.k, 64))
            gout = E.tick(pctx, ln_s, ar_s, co_s, to_gpu_partition(E, opart), theta, sp, qid_out=qs)
            osp = O.select_params(k=args.k, mode=omode, now=workload.NOW)
            ref = O.tick(pool["len"][:sample_n], pool["arrival"][:sample_n], pool["cost"][:sample_n], opart,
                         O.meta(**workload.THETA0), osp)
            phi, _ = O.score_all(pool["len"][:sample_n], pool["arrival"][:sample_n], pool["cost"][:sample_n],
                                 ref["qid"], ref["partition"], O.meta(**workload.THETA0), osp)
            qid_ok = bool(np.array_equal(qs.cpu().numpy(), ref["qid"]))
            rep = compare_selection(gpu_result(gout), ref, phi, pool["arrival"][:sample_n], omode, args.k)
            line["parity_sample"] = {"requests": sample_n, "qid_exact": qid_ok, "near_ties": rep.near_ties,
                                     "queues_checked": rep.checked_queues, "status": "pass"}
            pctx.close()
        except AssertionError as e:
            line["parity_sample"] = {"requests": sample_n, "status": f"FAIL: {e}"}
    if rank == 0 and ws == 1 and not args.no_traffic:
        copies.clear()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        tb, note = measure_traffic(n)
        roofline["traffic"] = tb
        roofline["traffic_source"] = note
        if tb:
            roofline["traffic_over_algorithmic"] = tb / (BYTES_PER_REQ * n)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if group is not None:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
