"""Thin torch-facing binding of libewsjf (argument marshalling only).

Every step of the path runs in the CUDA library; this module only turns torch
tensors into device pointers and ctypes structs.  Names follow the C ABI
(``ewsjf_tick`` -> ``tick`` ...).  See include/ewsjf.h for the contract.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib as L

__all__ = [
    "EwsjfError", "Context", "make_partition", "meta", "select_params", "partition_params", "weights_from_meta",
    "Outputs", "tick", "tick_host", "score_select", "route", "partition", "score_select_sweep", "meta_array",
    "exchange_bytes", "tick_local", "tick_merge", "tick_sharded", "batch_build", "prune_empty",
    "alloc_count", "history_hist", "partition_from_hist", "reduce_hist", "check_reduced", "partition_sharded", "online_adjust",
]


class EwsjfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"ewsjf status {status}: {msg}")
        self.status = status


def _ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


class Context:
    """Owns an ``ewsjf_ctx`` (all scratch preallocated for max_pool / max_history / max_k)."""

    def __init__(self, device: int = 0, max_pool: int = 0, max_history: int = 0, max_k: int = 64,
                 max_sweep: int = 0):
        self.lib = L.load()
        self.device = device
        self.max_k = max_k
        torch.cuda.init()
        h = C.c_void_p()
        with torch.cuda.device(device):
            st = torch.cuda.current_stream(device).cuda_stream
        s = self.lib.ewsjf_ctx_create(device, C.c_void_p(st), max_pool, max_history, max_k, C.byref(h))
        if s != L.OK:
            raise EwsjfError(s, "ewsjf_ctx_create failed")
        self.h = h
        if max_sweep > 0:      # Θ-sweep scratch reserved up front (the sweep call never allocates)
            self.check(self.lib.ewsjf_ctx_reserve_sweep(h, max_sweep), (L.OK,))

    @property
    def num_ctas(self) -> int:
        return self.lib.ewsjf_ctx_num_ctas(self.h)

    def use_current_stream(self):
        st = torch.cuda.current_stream(self.device).cuda_stream
        self.lib.ewsjf_ctx_set_stream(self.h, C.c_void_p(st))

    def set_timing(self, enable: bool = True):
        self.check(self.lib.ewsjf_ctx_set_timing(self.h, int(enable)))

    def timing(self) -> dict:
        t = L.Timing()
        self.check(self.lib.ewsjf_ctx_get_timing(self.h, C.byref(t)))
        return t.as_dict()

    def phases(self):
        """Per-CTA phase timestamps of the last streaming tick (EWSJF_PHASES), shape [ctas, 16]."""
        import numpy as np
        n = self.num_ctas * 32
        buf = (C.c_uint64 * n)()
        self.check(self.lib.ewsjf_ctx_get_phases(self.h, buf, n))
        return np.frombuffer(buf, dtype=np.uint64).reshape(self.num_ctas, 32).copy()

    def init_nccl(self, rank: int = 0, world: int = 1, group=None):
        """Give the ctx its own NCCL communicator (ewsjf_ctx_init_nccl): rank 0 creates
        the unique id in the library and it is broadcast over ``group`` (any
        torch.distributed backend; not needed at world 1).  From then on
        ``tick`` is the index-sharded tick of SURVEY §8e (NCCL all-gather inside
        the library)."""
        buf = (C.c_uint8 * L.NCCL_ID_BYTES)()
        if rank == 0:
            s = self.lib.ewsjf_nccl_get_unique_id(buf)
            if s != L.OK:
                raise EwsjfError(s, "ewsjf_nccl_get_unique_id (NCCL unavailable?)")
        if world > 1:
            import torch.distributed as dist
            obj = [bytes(buf) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            C.memmove(buf, obj[0], L.NCCL_ID_BYTES)
        self.check(self.lib.ewsjf_ctx_init_nccl(self.h, buf, rank, world), (L.OK,))
        self.nccl_world = world

    def ffma_rate(self) -> float:
        """Measured fp32 FFMA/s of the device (ewsjf_diag_ffma_rate)."""
        r = C.c_double(0.0)
        self.check(self.lib.ewsjf_diag_ffma_rate(self.h, C.byref(r)), (L.OK,))
        return r.value

    def set_exchange_gap_cap(self, gap_cap: int):
        """Gap entries per exchange record (ewsjf_ctx_set_exchange_gap_cap; default 1024)."""
        self.check(self.lib.ewsjf_ctx_set_exchange_gap_cap(self.h, int(gap_cap)), (L.OK,))

    def detach_nccl(self):
        self.check(self.lib.ewsjf_ctx_detach_nccl(self.h), (L.OK,))
        self.nccl_world = 0

    def check(self, s: int, allow=(L.OK, L.DOMAIN)) -> int:
        if s not in allow:
            msg = self.lib.ewsjf_last_error(self.h).decode()
            raise EwsjfError(s, msg or self.lib.ewsjf_status_str(s).decode())
        return s

    def close(self):
        if getattr(self, "h", None):
            self.lib.ewsjf_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- structs ---
def make_partition(bounds, means=None, ids=None, bubbles=None, counts=None, next_id=None) -> L.Partition:
    """Partition from [(min_len, max_len), ...] sorted and disjoint."""
    p = L.Partition()
    p.n = len(bounds)
    for i, (lo, hi) in enumerate(bounds):
        q = p.q[i]
        q.id = int(ids[i]) if ids is not None else i
        q.index = i + 1
        q.min_len, q.max_len = int(lo), int(hi)
        q.mean = float(means[i]) if means is not None else (lo + hi - 1) / 2.0
        q.is_bubble = int(bubbles[i]) if bubbles is not None else 0
        q.count = int(counts[i]) if counts is not None else 0
    p.next_id = next_id if next_id is not None else ((max(ids) + 1) if ids is not None and len(ids) else len(bounds))
    return p


def meta(a_b=0.0, b_b=1.0, a_u=-1e-4, b_u=2.0, a_f=1e-4, b_f=0.5) -> L.Meta:
    return L.Meta(a_b, b_b, a_u, b_u, a_f, b_f)


def select_params(k=64, mode=L.SELECT_SCORE, now=600.0, cost=(0.005, 0.0002, 1e-8)) -> L.SelectParams:
    return L.SelectParams(k, mode, now, L.CostParams(*cost))


def partition_params(alpha=2.0, min_width=1, max_queues=32, epsilon=1e-6, coarse_k=3, merge_rule=L.MIN_U,
                     gap_rule=0, kmeans_k=0):
    """kmeans_k > 0 selects the k-means-only partition (Table 3 "EWSJF (K-Means)")."""
    return L.PartitionParams(alpha, min_width, max_queues, epsilon, coarse_k, merge_rule, gap_rule, kmeans_k)


def alloc_count() -> int:
    """Process-wide count of the library's device/pinned allocations and frees."""
    return int(L.load().ewsjf_alloc_count())


def weights_from_meta(theta: L.Meta, part: L.Partition):
    w = (L.Weights * L.MAX_QUEUES)()
    s = L.load().ewsjf_weights_from_meta(C.byref(theta), C.byref(part), w)
    if s != L.OK:
        raise EwsjfError(s, "weights_from_meta")
    return w


@dataclass
class Outputs:
    """Device output buffers of a selection (rows = queue positions, MAX_QUEUES of them)."""
    topk_id: torch.Tensor
    topk_score: torch.Tensor
    count: torch.Tensor
    head_id: torch.Tensor
    head_score: torch.Tensor
    max_score: torch.Tensor
    summary_dev: torch.Tensor
    k: int
    summary: dict | None = None

    @staticmethod
    def alloc(k: int, device) -> "Outputs":
        Q = L.MAX_QUEUES
        return Outputs(
            torch.empty((Q, k), dtype=torch.int64, device=device), torch.empty((Q, k), dtype=torch.float32, device=device),
            torch.empty(Q, dtype=torch.int64, device=device), torch.empty(Q, dtype=torch.int64, device=device),
            torch.empty(Q, dtype=torch.float32, device=device), torch.empty(Q, dtype=torch.float32, device=device),
            torch.empty(C.sizeof(L.Summary), dtype=torch.uint8, device=device), k)

    def struct(self, h_summary=None) -> L.SelectOut:
        return L.SelectOut(self.topk_id.data_ptr(), self.topk_score.data_ptr(), self.count.data_ptr(),
                           self.head_id.data_ptr(), self.head_score.data_ptr(), self.max_score.data_ptr(),
                           self.summary_dev.data_ptr(), C.pointer(h_summary) if h_summary is not None else None)

    def nq(self) -> int:
        return self.summary["n_queues"]

    def fetch_summary(self) -> dict:
        """Copy the device summary of an asynchronous call (e.g. one Θ of a sweep) to the host."""
        b = bytes(self.summary_dev.cpu().numpy().tobytes())
        self.summary = L.Summary.from_buffer_copy(b).as_dict()
        return self.summary


def _dev_check(t: torch.Tensor | None, dtype, name):
    if t is None:
        return
    if not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous CUDA {dtype} tensor")


# --------------------------------------------------------------- tactical ---
def tick(ctx: Context, length, arrival, cost, part: L.Partition, theta: L.Meta, params: L.SelectParams,
         bubble_width: int = 64, global_base: int = 0, qid_out=None, out: Outputs | None = None,
         sync: bool = True) -> Outputs:
    """ewsjf_tick: route + bubbles + weights + score + per-queue selection over the pool."""
    _dev_check(length, torch.int32, "len"); _dev_check(arrival, torch.float32, "arrival")
    _dev_check(cost, torch.float32, "cost"); _dev_check(qid_out, torch.int32, "qid_out")
    out = out or Outputs.alloc(params.k, length.device)
    ctx.use_current_stream()
    hs = L.Summary() if sync else None
    so = out.struct(hs)
    s = ctx.lib.ewsjf_tick(ctx.h, _ptr(length), _ptr(arrival), _ptr(cost), length.numel(), global_base,
                           C.byref(part), bubble_width, C.byref(theta), C.byref(params), _ptr(qid_out), C.byref(so))
    ctx.check(s, (L.OK, L.DOMAIN, L.CAPACITY))
    out.summary = hs.as_dict() if sync else None
    return out


def tick_host(ctx: Context, length, arrival, cost, part: L.Partition, theta: L.Meta, params: L.SelectParams,
              bubble_width: int = 64, global_base: int = 0, qid_out=None, results=None) -> dict:
    """ewsjf_tick_host: host (pinned) buffers in, host results out; H2D/D2H inside the call."""
    n = length.numel()
    K = params.k
    Q = L.MAX_QUEUES
    r = results or {
        "topk_id": torch.empty((Q, K), dtype=torch.int64).pin_memory(),
        "topk_score": torch.empty((Q, K), dtype=torch.float32).pin_memory(),
        "count": torch.empty(Q, dtype=torch.int64).pin_memory(),
        "head_id": torch.empty(Q, dtype=torch.int64).pin_memory(),
        "head_score": torch.empty(Q, dtype=torch.float32).pin_memory(),
        "max_score": torch.empty(Q, dtype=torch.float32).pin_memory(),
    }
    hs = L.Summary()
    ctx.use_current_stream()
    s = ctx.lib.ewsjf_tick_host(ctx.h, _ptr(length), _ptr(arrival), _ptr(cost), n, global_base, C.byref(part),
                                bubble_width, C.byref(theta), C.byref(params), _ptr(qid_out),
                                _ptr(r["topk_id"]), _ptr(r["topk_score"]), _ptr(r["count"]), _ptr(r["head_id"]),
                                _ptr(r["head_score"]), _ptr(r["max_score"]), C.byref(hs))
    ctx.check(s, (L.OK, L.DOMAIN, L.CAPACITY))
    r["summary"] = hs.as_dict()
    return r


def score_select(ctx: Context, length, arrival, cost, qid, part: L.Partition, weights, params: L.SelectParams,
                 out: Outputs | None = None, sync: bool = True) -> Outputs:
    """ewsjf_score_select over an already routed pool (weights by queue position)."""
    _dev_check(length, torch.int32, "len"); _dev_check(arrival, torch.float32, "arrival")
    _dev_check(cost, torch.float32, "cost"); _dev_check(qid, torch.int32, "qid")
    out = out or Outputs.alloc(params.k, length.device)
    ctx.use_current_stream()
    hs = L.Summary() if sync else None
    so = out.struct(hs)
    s = ctx.lib.ewsjf_score_select(ctx.h, _ptr(length), _ptr(arrival), _ptr(cost), _ptr(qid), length.numel(),
                                   C.byref(part), weights, C.byref(params), C.byref(so))
    ctx.check(s, (L.OK, L.DOMAIN, L.CAPACITY))
    out.summary = hs.as_dict() if sync else None
    return out


def route(ctx: Context, length, part: L.Partition, bubble_width: int = 64, qid_out=None):
    """ewsjf_route: stable queue id per request; bubbles are inserted into ``part``."""
    _dev_check(length, torch.int32, "len")
    qid = qid_out if qid_out is not None else torch.empty_like(length)
    ctx.use_current_stream()
    hs = L.Summary()
    s = ctx.lib.ewsjf_route(ctx.h, _ptr(length), length.numel(), C.byref(part), bubble_width, _ptr(qid), C.byref(hs))
    ctx.check(s, (L.OK, L.DOMAIN, L.CAPACITY))
    return qid, hs.as_dict()


def partition(ctx: Context, length, params: L.PartitionParams | None = None):
    """ewsjf_partition: Refine-and-Prune over a device history.  Returns (Partition, stats dict, status)."""
    _dev_check(length, torch.int32, "len")
    params = params or partition_params()
    ctx.use_current_stream()
    out = L.Partition()
    st = L.PartitionStats()
    s = ctx.lib.ewsjf_partition(ctx.h, _ptr(length), length.numel(), C.byref(params), C.byref(out), C.byref(st))
    ctx.check(s, (L.OK, L.DOMAIN, L.EMPTY))
    return out, {f: getattr(st, f) for f, _ in L.PartitionStats._fields_}, s


def history_hist(ctx: Context, length, hist_out=None):
    """ewsjf_history_hist: A1 histogram of a device history (int32 view of the uint32
    bins, HIST_BINS + 1 entries).  Returns (hist, {"invalid", "over", "max_len"}).

    Lengths >= HIST_BINS do not raise here (status UNSUPPORTED, counted in
    "over"): in a sharded run every rank must still enter the all-reduce, and
    all of them then refuse together (``check_reduced``)."""
    _dev_check(length, torch.int32, "len")
    hist = hist_out if hist_out is not None else torch.empty(L.HIST_BINS + 1, dtype=torch.int32, device=length.device)
    _dev_check(hist, torch.int32, "hist_out")
    info = (C.c_int64 * 3)()
    ctx.use_current_stream()
    s = ctx.lib.ewsjf_history_hist(ctx.h, _ptr(length), length.numel(), _ptr(hist), info)
    ctx.check(s, (L.OK, L.UNSUPPORTED))
    return hist, {"invalid": info[0], "over": info[1], "max_len": info[2]}


def check_reduced(info: dict):
    """After reduce_hist: every rank raises together if any shard held a length
    the histogram cannot bin (the summed "over" count is identical on all ranks)."""
    if info["over"] > 0:
        raise EwsjfError(L.UNSUPPORTED, f"{info['over']} history lengths >= {L.HIST_BINS} across the shards")


def partition_from_hist(ctx: Context, hist, max_len: int, n_invalid: int = 0,
                        params: L.PartitionParams | None = None):
    """ewsjf_partition_from_hist: A2..A6 from a (summed) histogram -> (Partition, stats, status)."""
    _dev_check(hist, torch.int32, "hist")
    params = params or partition_params()
    ctx.use_current_stream()
    out = L.Partition()
    st = L.PartitionStats()
    s = ctx.lib.ewsjf_partition_from_hist(ctx.h, _ptr(hist), max_len, n_invalid, C.byref(params), C.byref(out),
                                          C.byref(st))
    ctx.check(s, (L.OK, L.DOMAIN, L.EMPTY))
    return out, {f: getattr(st, f) for f, _ in L.PartitionStats._fields_}, s


def online_adjust(ctx: Context, window, part: L.Partition, max_shift: float = 0.25) -> int:
    """ewsjf_online_adjust: bounded local-quantile boundary shifts from a recent
    window (device int32 lengths); updates ``part`` in place, returns boundaries moved."""
    _dev_check(window, torch.int32, "window")
    ctx.use_current_stream()
    mv = C.c_int32(0)
    s = ctx.lib.ewsjf_online_adjust(ctx.h, _ptr(window), window.numel(), max_shift, C.byref(part), C.byref(mv))
    ctx.check(s, (L.OK,))
    return mv.value


def reduce_hist(hist, info: dict, group=None):
    """All-reduce of the ranks' histograms (exact integer SUM) and of their A1
    statistics (invalid: SUM, max_len: MAX) over ``group`` — in place on ``hist``."""
    import torch.distributed as dist
    dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    t = torch.tensor([info["invalid"], info["over"]], dtype=torch.int64, device=hist.device)
    m = torch.tensor([info["max_len"]], dtype=torch.int64, device=hist.device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    return hist, {"invalid": int(t[0]), "over": int(t[1]), "max_len": int(m[0])}


def partition_sharded(ctx: Context, length_shard, params: L.PartitionParams | None = None, group=None):
    """Refine-and-Prune of a history sharded across the ranks of ``group`` (NCCL):
    local histogram, all-reduce, A2..A6 on every rank (identical, replicated result)."""
    hist, info = history_hist(ctx, length_shard)
    hist, info = reduce_hist(hist, info, group)      # every rank, even one that saw an over-long length
    check_reduced(info)
    return partition_from_hist(ctx, hist, info["max_len"], info["invalid"], params)


_SWEEP_OUT_CACHE: dict = {}


def meta_array(thetas: list[L.Meta]):
    """A ctypes array of Θ for score_select_sweep (built once, reused across calls)."""
    return (L.Meta * len(thetas))(*thetas)


def score_select_sweep(ctx: Context, length, arrival, cost, qid, part: L.Partition, thetas: list[L.Meta],
                       params: L.SelectParams, outs: list[Outputs] | None = None) -> list[Outputs]:
    """ewsjf_score_select_sweep: one selection per Θ over one routed snapshot (A12)."""
    n_theta = len(thetas)
    outs = outs or [Outputs.alloc(params.k, length.device) for _ in range(n_theta)]
    # thetas may be a prebuilt ctypes array (meta_array): no per-call conversion
    th = thetas if isinstance(thetas, C.Array) else (L.Meta * n_theta)(*thetas)
    # the output descriptor array of a given list of Outputs is built once (their tensors
    # are fixed at allocation); building 256 of them per call took ~1 ms of host time
    key = tuple(map(id, outs))
    so = _SWEEP_OUT_CACHE.get(key)
    if so is None or so[0] is not outs[0]:
        so = (outs[0], (L.SelectOut * n_theta)(*[o.struct() for o in outs]))
        _SWEEP_OUT_CACHE.clear()
        _SWEEP_OUT_CACHE[key] = so
    so = so[1]
    ctx.use_current_stream()
    s = ctx.lib.ewsjf_score_select_sweep(ctx.h, _ptr(length), _ptr(arrival), _ptr(cost), _ptr(qid), length.numel(),
                                         C.byref(part), th, n_theta, C.byref(params), so)
    ctx.check(s, (L.OK, L.DOMAIN))
    return outs


# ------------------------------------------------------ Alg. 1 batch ------
def batch_build(ctx: Context, length, sel: Outputs, n_queues: int, max_requests: int, max_tokens: int,
                global_base: int = 0, ids_out=None, info_out=None):
    """ewsjf_batch_build over a FIFO-mode selection ``sel`` (depth >= max_requests).

    Returns (ids [max_requests] int64 device, -1 padded; info [4] int64 device:
    count, tokens, status, primary).  Asynchronous on the current stream."""
    _dev_check(length, torch.int32, "len")
    ids = ids_out if ids_out is not None else torch.empty(max_requests, dtype=torch.int64, device=length.device)
    info = info_out if info_out is not None else torch.empty(4, dtype=torch.int64, device=length.device)
    _dev_check(ids, torch.int64, "ids_out"); _dev_check(info, torch.int64, "info_out")
    so = sel.struct()
    b = L.Budget(max_requests, 0, max_tokens)
    ctx.use_current_stream()
    s = ctx.lib.ewsjf_batch_build(ctx.h, _ptr(length), length.numel(), global_base, C.byref(so), sel.k,
                                  n_queues, C.byref(b), _ptr(ids), _ptr(info))
    ctx.check(s, (L.OK,))
    return ids, info


def prune_empty(part: L.Partition, counts, threshold: int) -> int:
    """ewsjf_prune_empty (host): Alg. 1 lines 8-12 on ``part`` in place; returns queues removed."""
    import numpy as np
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.int64)[: part.n])
    rm = C.c_int32(0)
    s = L.load().ewsjf_prune_empty(C.byref(part), c.ctypes.data, threshold, C.byref(rm))
    if s != L.OK:
        raise RuntimeError(f"ewsjf_prune_empty: status {s}")
    return rm.value


# ----------------------------------------------------------- multi-GPU ------
def exchange_bytes(ctx: Context, n_queues: int, k: int) -> int:
    return int(ctx.lib.ewsjf_exchange_bytes(ctx.h, n_queues, k))


def tick_local(ctx: Context, length, arrival, cost, global_base: int, part, theta, params, qid_out=None,
               exchange: torch.Tensor | None = None) -> torch.Tensor:
    nb = exchange_bytes(ctx, part.n, params.k)
    ex = exchange if exchange is not None else torch.empty(nb, dtype=torch.uint8, device=length.device)
    ctx.use_current_stream()
    s = ctx.lib.ewsjf_tick_local(ctx.h, _ptr(length), _ptr(arrival), _ptr(cost), length.numel(), global_base,
                                 C.byref(part), C.byref(theta), C.byref(params), _ptr(qid_out), ex.data_ptr())
    ctx.check(s)
    return ex


def tick_merge(ctx: Context, exchange_all: torch.Tensor, world: int, global_base: int, n_local: int, qid_local,
               part, theta, params, bubble_width: int = 64, out: Outputs | None = None, sync: bool = True) -> Outputs:
    out = out or Outputs.alloc(params.k, exchange_all.device)
    ctx.use_current_stream()
    hs = L.Summary() if sync else None
    so = out.struct(hs)
    s = ctx.lib.ewsjf_tick_merge(ctx.h, exchange_all.data_ptr(), world, global_base, n_local, _ptr(qid_local),
                                 C.byref(part), bubble_width, C.byref(theta), C.byref(params), C.byref(so))
    ctx.check(s, (L.OK, L.DOMAIN, L.CAPACITY))
    out.summary = hs.as_dict() if sync else None
    return out


def tick_sharded(ctx: Context, length, arrival, cost, global_base: int, part, theta, params, group=None,
                 bubble_width: int = 64, qid_out=None, out: Outputs | None = None, sync: bool = True) -> Outputs:
    """Sharded tick: local route/score/reduce -> all-gather of the fixed-size
    exchange records over the process group (NCCL over NVLink) -> replicated global merge."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    ex = tick_local(ctx, length, arrival, cost, global_base, part, theta, params, qid_out)
    allx = torch.empty(world * ex.numel(), dtype=torch.uint8, device=ex.device)
    dist.all_gather_into_tensor(allx, ex, group=group)
    return tick_merge(ctx, allx, world, global_base, length.numel(), qid_out, part, theta, params,
                      bubble_width, out, sync)
