"""CPU oracle for libewsjf — TEST INFRASTRUCTURE ONLY.

Plain fp64 C (``ewsjf_oracle.c``) of what PAPER.md (arXiv 2601.21758) defines
for the scheduling tick and Refine-and-Prune, wrapped with ctypes.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA product (``paper_2601_21758_b200``) and never imports it.

Every function documents the passage it follows; see ``ewsjf_oracle.h``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ewsjf_oracle.c")
_LIB = os.path.join(_HERE, "libewsjf_oracle.so")

MAXQ = 256
OK, INVALID, DOMAIN, EMPTY, CAPACITY = 0, 1, 2, 3, 4
MIN_U, MAX_U = 0, 1
SCORE, FIFO = 0, 1


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -ffp-contract=off: no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "ewsjf_oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
             "-shared", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


class Queue(C.Structure):
    _fields_ = [
        ("id", C.c_int32), ("index", C.c_int32), ("min_len", C.c_int32), ("max_len", C.c_int32),
        ("count", C.c_int64), ("sum", C.c_int64), ("sumsq", C.c_int64),
        ("mean", C.c_double), ("density", C.c_double), ("sse", C.c_double),
        ("is_bubble", C.c_int32), ("pad", C.c_int32),
    ]


class Partition(C.Structure):
    _fields_ = [("n", C.c_int32), ("next_id", C.c_int32), ("q", Queue * MAXQ)]

    def queues(self) -> list[dict]:
        out = []
        for i in range(self.n):
            q = self.q[i]
            out.append({f: getattr(q, f) for f, _ in Queue._fields_ if f != "pad"})
        return out


class Params(C.Structure):
    _fields_ = [("alpha", C.c_double), ("min_width", C.c_int32), ("max_queues", C.c_int32),
                ("epsilon", C.c_double), ("coarse_k", C.c_int32), ("merge_rule", C.c_int32),
                ("gap_rule", C.c_int32)]


class PartitionStats(C.Structure):
    _fields_ = [("n_valid", C.c_int64), ("n_invalid", C.c_int64), ("distinct", C.c_int64),
                ("k_used", C.c_int32), ("t1", C.c_int32), ("t2", C.c_int32),
                ("segments", C.c_int64), ("depth", C.c_int32), ("merges", C.c_int64)]


class Meta(C.Structure):
    _fields_ = [(f, C.c_double) for f in ("a_b", "b_b", "a_u", "b_u", "a_f", "b_f")]


class SelectParams(C.Structure):
    _fields_ = [("k", C.c_int32), ("mode", C.c_int32), ("now", C.c_float),
                ("c0", C.c_float), ("c1", C.c_float), ("c2", C.c_float)]


class SelectOut(C.Structure):
    _fields_ = [
        ("topk_id", C.POINTER(C.c_int64)), ("topk_score", C.POINTER(C.c_double)),
        ("count", C.POINTER(C.c_int64)), ("head_id", C.POINTER(C.c_int64)),
        ("head_score", C.POINTER(C.c_double)), ("max_score", C.POINTER(C.c_double)),
        ("primary", C.c_int32), ("n_excluded", C.c_int64), ("n_invalid", C.c_int64),
        ("n_bubbles", C.c_int64), ("n_dropped", C.c_int64),
    ]


_lib = None


class Budget(C.Structure):
    _fields_ = [("max_requests", C.c_int32), ("max_tokens", C.c_int64)]


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER
        L = _lib
        L.or_rle.restype = C.c_int64
        L.or_rle.argtypes = [P(C.c_int32), C.c_int64, P(C.c_int32), P(C.c_int64), P(C.c_int64)]
        L.or_prefix.argtypes = [P(C.c_int32), P(C.c_int64), C.c_int64, P(C.c_int64), P(C.c_int64), P(C.c_int64)]
        L.or_kmeans.argtypes = [P(C.c_int64), P(C.c_int64), C.c_int64, C.c_int32, P(C.c_int32)]
        L.or_kmeans_dp.argtypes = [P(C.c_int64), P(C.c_int64), C.c_int64, C.c_int32, P(C.c_int32)]
        L.or_partition_kmeans.argtypes = [P(C.c_int32), C.c_int64, C.c_int32, P(Partition), P(PartitionStats)]
        L.or_refine.restype = C.c_int64
        L.or_refine.argtypes = [P(C.c_int32), P(C.c_int64), C.c_int64, C.c_int64, C.c_double, C.c_int32,
                                P(C.c_int64), P(C.c_int32)]
        L.or_utility.restype = C.c_double
        L.or_utility.argtypes = [C.c_double] * 5
        L.or_partition_run.argtypes = [P(C.c_int32), C.c_int64, P(Params), P(Partition), P(PartitionStats)]
        L.or_prune.restype = C.c_int64
        L.or_prune.argtypes = [C.c_int64, P(C.c_int32), P(C.c_int32), P(C.c_int64), P(C.c_int64), P(C.c_int64),
                               C.c_int32, C.c_double, C.c_int32, P(C.c_int64)]
        L.or_weights.argtypes = [P(Meta), C.c_double, P(C.c_float)]
        L.or_route.argtypes = [P(C.c_int32), C.c_int64, P(Partition), C.c_int32, P(C.c_int32),
                               P(C.c_int64), P(C.c_int64), P(C.c_int64)]
        L.or_score_one.argtypes = [C.c_int32, C.c_float, P(C.c_float), C.c_int32, P(C.c_float),
                                   P(SelectParams), P(C.c_double)]
        L.or_score_select.argtypes = [P(C.c_int32), P(C.c_float), P(C.c_float), P(C.c_int32), C.c_int64,
                                      C.c_int64, P(Partition), P(C.c_float), P(SelectParams), P(SelectOut)]
        L.or_score_all.argtypes = [P(C.c_int32), P(C.c_float), P(C.c_float), P(C.c_int32), C.c_int64, P(Partition),
                                   P(C.c_float), P(SelectParams), P(C.c_double), P(C.c_int8)]
        L.or_tick.argtypes = [P(C.c_int32), P(C.c_float), P(C.c_float), C.c_int64, C.c_int64, P(Partition),
                              C.c_int32, P(Meta), P(SelectParams), P(C.c_int32), P(SelectOut)]
        L.or_sweep.argtypes = [P(C.c_int32), P(C.c_float), P(C.c_float), P(C.c_int32), C.c_int64, C.c_int64,
                               P(Partition), P(Meta), C.c_int32, P(SelectParams), P(SelectOut)]
        L.or_batch.restype = C.c_int64
        L.or_batch.argtypes = [P(C.c_int32), P(C.c_float), P(C.c_float), P(C.c_int32), C.c_int64, C.c_int64,
                               P(Partition), P(SelectParams), C.c_int32, P(Budget), P(C.c_int64), P(C.c_int64)]
        L.or_prune_empty.restype = C.c_int32
        L.or_prune_empty.argtypes = [P(Partition), P(C.c_int32), P(C.c_int64), C.c_int32]
        L.or_online_adjust.restype = C.c_int32
        L.or_online_adjust.argtypes = [P(C.c_int32), C.c_int64, C.c_double, P(Partition)]
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.int32)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.float32)


# ---------------------------------------------------------------- partition ---
def rle(lengths):
    """O1: sorted RLE (v, c) of the history and #invalid (< 1)."""
    x = _i32(lengths)
    n = len(x)
    v = np.zeros(max(n, 1), np.int32)
    c = np.zeros(max(n, 1), np.int64)
    bad = C.c_int64()
    M = lib().or_rle(_p(x, C.c_int32), n, _p(v, C.c_int32), _p(c, C.c_int64), C.byref(bad))
    return v[:M].copy(), c[:M].copy(), bad.value


def prefix(v, c):
    """O2: int64 prefix sums N, S1, S2 over the RLE."""
    v = _i32(v); c = np.ascontiguousarray(c, dtype=np.int64)
    M = len(v)
    N = np.zeros(M + 1, np.int64); S1 = np.zeros(M + 1, np.int64); S2 = np.zeros(M + 1, np.int64)
    lib().or_prefix(_p(v, C.c_int32), _p(c, C.c_int64), M, _p(N, C.c_int64), _p(S1, C.c_int64), _p(S2, C.c_int64))
    return N, S1, S2


def kmeans(lengths, k):
    """O3: exact 1-D k-means (k <= 3) of a multiset; returns the clusters as lists
    of values (SPEC kmeans_1d shape)."""
    v, c, _ = rle(lengths)
    N, S1, _ = prefix(v, c)
    cuts = np.zeros(2, np.int32)
    st = lib().or_kmeans(_p(N, C.c_int64), _p(S1, C.c_int64), len(v), k, _p(cuts, C.c_int32))
    if st != OK:
        raise ValueError("k out of range")
    b = [0] + [int(t) for t in cuts[: k - 1]] + [len(v)]
    return [sorted(np.repeat(v[b[i]:b[i + 1]], c[b[i]:b[i + 1]]).tolist()) for i in range(k)]


def kmeans_dp(lengths, k):
    """O14: exact 1-D k-means for any k (DP, R32); the clusters as sorted value lists."""
    v, c, _ = rle(lengths)
    N, S1, _ = prefix(v, c)
    ku = min(k, len(v))
    cuts = np.zeros(max(ku, 1), np.int32)
    st = lib().or_kmeans_dp(_p(N, C.c_int64), _p(S1, C.c_int64), len(v), k, _p(cuts, C.c_int32))
    if st != OK:
        raise ValueError("k out of range")
    b = [0] + [int(t) for t in cuts[: ku - 1]] + [len(v)]
    return [sorted(np.repeat(v[b[i]:b[i + 1]], c[b[i]:b[i + 1]]).tolist()) for i in range(ku)]


def partition_kmeans(lengths, k):
    """O14 partition: k-means-only queues with O5's finalisation (Table 3 "EWSJF (K-Means)").
    Returns (status, Partition, stats)."""
    x = _i32(lengths)
    part = Partition()
    st = PartitionStats()
    s = lib().or_partition_kmeans(_p(x, C.c_int32), len(x), k, C.byref(part), C.byref(st))
    return s, part, st


def refine(values, alpha, min_width=1):
    """O4 on one cluster (SPEC refine_cluster): list of sub-clusters."""
    v, c, _ = rle(values)
    N, _, _ = prefix(v, c)
    seg = np.zeros(len(v) + 1, np.int64)
    depth = C.c_int32(0)
    m = lib().or_refine(_p(v, C.c_int32), _p(N, C.c_int64), 0, len(v), alpha, min_width,
                        _p(seg, C.c_int64), C.byref(depth))
    starts = seg[:m].tolist() + [len(v)]
    return [np.repeat(v[starts[i]:starts[i + 1]], c[starts[i]:starts[i + 1]]).tolist() for i in range(m)]


def utility(rho_l, rho_r, mean_l, mean_r, eps):
    """Eq. 3 for one adjacent pair."""
    return lib().or_utility(rho_l, rho_r, mean_l, mean_r, eps)


def prune(lo, hi, cnt, s1, s2, max_queues, eps, rule=MIN_U):
    """O6 on explicit candidate queues; returns (lo, hi, cnt, s1, s2, merges)."""
    lo = _i32(lo).copy(); hi = _i32(hi).copy()
    cnt = np.array(cnt, np.int64); s1 = np.array(s1, np.int64); s2 = np.array(s2, np.int64)
    merges = C.c_int64()
    m = lib().or_prune(len(lo), _p(lo, C.c_int32), _p(hi, C.c_int32), _p(cnt, C.c_int64), _p(s1, C.c_int64),
                       _p(s2, C.c_int64), max_queues, eps, rule, C.byref(merges))
    return lo[:m], hi[:m], cnt[:m], s1[:m], s2[:m], merges.value


def params(alpha=2.0, min_width=1, max_queues=32, epsilon=1e-6, coarse_k=3, merge_rule=MIN_U, gap_rule=0) -> Params:
    return Params(alpha, min_width, max_queues, epsilon, coarse_k, merge_rule, gap_rule)


def partition(lengths, **kw):
    """O1..O6: Refine-and-Prune (§4.2).  Returns (status, Partition, stats)."""
    x = _i32(lengths)
    part = Partition()
    st = PartitionStats()
    p = params(**kw)
    s = lib().or_partition_run(_p(x, C.c_int32), len(x), C.byref(p), C.byref(part), C.byref(st))
    return s, part, st


def make_partition(bounds, means=None, ids=None, bubbles=None) -> Partition:
    """Build a Partition from [(min_len, max_len), ...] (sorted, disjoint)."""
    part = Partition()
    part.n = len(bounds)
    for i, (lo, hi) in enumerate(bounds):
        q = part.q[i]
        q.id = ids[i] if ids is not None else i
        q.index = i + 1
        q.min_len, q.max_len = int(lo), int(hi)
        q.mean = float(means[i]) if means is not None else (lo + hi - 1) / 2.0
        q.density = 0.0
        q.is_bubble = int(bubbles[i]) if bubbles is not None else 0
    part.next_id = (max(ids) + 1) if ids is not None and len(ids) else len(bounds)
    return part


def copy_partition(part: Partition) -> Partition:
    out = Partition()
    C.memmove(C.byref(out), C.byref(part), C.sizeof(Partition))
    return out


# ------------------------------------------------------------------ tactical ---
def meta(a_b=0.0, b_b=1.0, a_u=-1e-4, b_u=2.0, a_f=1e-4, b_f=0.5) -> Meta:
    return Meta(a_b, b_b, a_u, b_u, a_f, b_f)


def weights(theta: Meta, mean: float):
    """O7: (w_base, w_urg, w_fair) as fp32."""
    w = (C.c_float * 3)()
    lib().or_weights(C.byref(theta), mean, w)
    return np.array(list(w), np.float32)


def route(lengths, part: Partition, bubble_width: int):
    """O8 (Alg. 2). Mutates ``part``.  Returns (status, qid, n_invalid, n_bubbles, n_dropped)."""
    x = _i32(lengths)
    qid = np.zeros(max(len(x), 1), np.int32)
    a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
    s = lib().or_route(_p(x, C.c_int32), len(x), C.byref(part), bubble_width, _p(qid, C.c_int32),
                       C.byref(a), C.byref(b), C.byref(c))
    return s, qid[: len(x)], a.value, b.value, c.value


def select_params(k=64, mode=SCORE, now=600.0, c0=0.005, c1=0.0002, c2=1e-8) -> SelectParams:
    return SelectParams(k, mode, now, c0, c1, c2)


def score_one(b, arrival, index, w, sp: SelectParams, cost=None):
    """O9: Eq. 4 in fp64 for one request; None if excluded."""
    wf = _f32(w)
    phi = C.c_double()
    cp = C.byref(C.c_float(cost)) if cost is not None else None
    r = lib().or_score_one(int(b), float(arrival), cp, int(index), _p(wf, C.c_float), C.byref(sp), C.byref(phi))
    return None if r else phi.value


class _Outs:
    def __init__(self, nq, k):
        self.topk_id = np.full(nq * k, -1, np.int64)
        self.topk_score = np.zeros(nq * k, np.float64)
        self.count = np.zeros(nq, np.int64)
        self.head_id = np.zeros(nq, np.int64)
        self.head_score = np.zeros(nq, np.float64)
        self.max_score = np.zeros(nq, np.float64)
        self.s = SelectOut(_p(self.topk_id, C.c_int64), _p(self.topk_score, C.c_double),
                           _p(self.count, C.c_int64), _p(self.head_id, C.c_int64),
                           _p(self.head_score, C.c_double), _p(self.max_score, C.c_double), -1, 0, 0, 0, 0)

    def result(self, nq, k, status, part):
        return {
            "status": status, "nq": nq, "k": k,
            "topk_id": self.topk_id[: nq * k].reshape(nq, k), "topk_score": self.topk_score[: nq * k].reshape(nq, k),
            "count": self.count[:nq], "head_id": self.head_id[:nq], "head_score": self.head_score[:nq],
            "max_score": self.max_score[:nq], "primary": self.s.primary,
            "n_excluded": self.s.n_excluded, "n_invalid": self.s.n_invalid,
            "n_bubbles": self.s.n_bubbles, "n_dropped": self.s.n_dropped,
            "partition": part,
        }


def score_select(lengths, arrival, cost, qid, part: Partition, w, sp: SelectParams, global_base=0):
    """O9 + O10 over an already routed pool; ``w`` is [nq, 3] by position."""
    x = _i32(lengths); a = _f32(arrival); q = _i32(qid)
    cst = _f32(cost) if cost is not None else None
    wf = _f32(w).reshape(-1)
    o = _Outs(part.n, sp.k)
    s = lib().or_score_select(_p(x, C.c_int32), _p(a, C.c_float), _p(cst, C.c_float) if cst is not None else None,
                              _p(q, C.c_int32), len(x), global_base, C.byref(part), _p(wf, C.c_float),
                              C.byref(sp), C.byref(o.s))
    return o.result(part.n, sp.k, s, part)


def sweep(lengths, arrival, cost, qid, part: Partition, thetas, sp: SelectParams, global_base=0):
    """O11: O7 -> O9 -> O10 per Θ over one routed snapshot; returns (status, [result per Θ])."""
    x = _i32(lengths); a = _f32(arrival); q = _i32(qid)
    cst = _f32(cost) if cost is not None else None
    outs = [_Outs(part.n, sp.k) for _ in thetas]
    thetas = [t if isinstance(t, Meta) else meta(**t) for t in thetas]
    arr = (Meta * max(1, len(thetas)))(*thetas)
    so = (SelectOut * max(1, len(thetas)))(*[o.s for o in outs])
    s = lib().or_sweep(_p(x, C.c_int32), _p(a, C.c_float), _p(cst, C.c_float) if cst is not None else None,
                       _p(q, C.c_int32), len(x), global_base, C.byref(part), arr, len(thetas), C.byref(sp), so)
    res = []
    for t, o in enumerate(outs):
        o.s = so[t]
        res.append(o.result(part.n, sp.k, s, part))
    return s, res


def score_all(lengths, arrival, cost, qid, part: Partition, theta: Meta, sp: SelectParams):
    """O9 for every request of a routed pool with weights O7(theta, queue mean): (phi, valid)."""
    x = _i32(lengths); a = _f32(arrival); q = _i32(qid)
    cst = _f32(cost) if cost is not None else None
    w = np.concatenate([weights(theta, part.q[i].mean) for i in range(part.n)] or [np.zeros(0, np.float32)])
    w = _f32(w)
    phi = np.zeros(max(len(x), 1), np.float64)
    valid = np.zeros(max(len(x), 1), np.int8)
    lib().or_score_all(_p(x, C.c_int32), _p(a, C.c_float), _p(cst, C.c_float) if cst is not None else None,
                       _p(q, C.c_int32), len(x), C.byref(part), _p(w, C.c_float) if len(w) else None,
                       C.byref(sp), _p(phi, C.c_double), _p(valid, C.c_int8))
    return phi[: len(x)], valid[: len(x)].astype(bool)


def tick(lengths, arrival, cost, part: Partition, theta: Meta, sp: SelectParams, bubble_width=64, global_base=0):
    """O8 + O7 + O9 + O10 (Alg. 1 + App. D over the whole pool).  ``part`` is copied, not mutated."""
    x = _i32(lengths); a = _f32(arrival)
    cst = _f32(cost) if cost is not None else None
    p2 = copy_partition(part)
    qid = np.zeros(max(len(x), 1), np.int32)
    o = _Outs(MAXQ, sp.k)
    s = lib().or_tick(_p(x, C.c_int32), _p(a, C.c_float), _p(cst, C.c_float) if cst is not None else None,
                      len(x), global_base, C.byref(p2), bubble_width, C.byref(theta), C.byref(sp),
                      _p(qid, C.c_int32), C.byref(o.s))
    res = o.result(p2.n, sp.k, s, p2)
    res["qid"] = qid[: len(x)]
    return res


def batch(lengths, arrival, cost, qid, part: Partition, sp: SelectParams, primary: int, max_requests: int,
          max_tokens: int, global_base=0):
    """O12: Alg. 1's Batch Builder (GreedyFill + Backfill) over a routed pool -> (ids, tokens)."""
    x = _i32(lengths); a = _f32(arrival); q = _i32(qid)
    cst = _f32(cost) if cost is not None else None
    ids = np.full(max(max_requests, 1), -1, np.int64)
    tok = C.c_int64(0)
    b = Budget(max_requests, max_tokens)
    nb = lib().or_batch(_p(x, C.c_int32), _p(a, C.c_float), _p(cst, C.c_float) if cst is not None else None,
                        _p(q, C.c_int32), len(x), global_base, C.byref(part), C.byref(sp), primary, C.byref(b),
                        _p(ids, C.c_int64), C.byref(tok))
    return ids[:nb], tok.value


def prune_empty(part: Partition, empty_cnt, counts, threshold: int):
    """Alg. 1 lines 8-12 on a copy of ``part``: (new partition, new empty counters, removed)."""
    p2 = copy_partition(part)
    e = np.ascontiguousarray(np.asarray(empty_cnt, np.int32).copy())
    c = np.ascontiguousarray(np.asarray(counts, np.int64))
    removed = lib().or_prune_empty(C.byref(p2), _p(e, C.c_int32), _p(c, C.c_int64), threshold)
    return p2, e[: p2.n], removed


def online_adjust(window, part: Partition, max_shift: float = 0.25):
    """O13: online adjust (R31) on a copy of ``part`` -> (new partition, boundaries moved)."""
    w = _i32(window)
    p2 = copy_partition(part)
    moved = lib().or_online_adjust(_p(w, C.c_int32), len(w), max_shift, C.byref(p2))
    return p2, moved
