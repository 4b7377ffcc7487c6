"""GPU-vs-oracle comparators (test helpers; import only from tests).

Bar (north_star / SURVEY §8c): bit-exact for integer work (qids, counts,
FIFO ids, head ids, partition bounds); fp32 scores within 1e-5 relative of the
fp64 oracle; SCORE-mode ids exact except at near-ties (|ΔΦ| <= 1e-5 relative).
"""
from __future__ import annotations

import numpy as np

REL = 1e-5


def to_gpu_partition(E, opart):
    """Oracle Partition -> libewsjf Partition with identical bounds / ids / means / stats."""
    qs = opart.queues()
    p = E.make_partition([(q["min_len"], q["max_len"]) for q in qs], means=[q["mean"] for q in qs],
                         ids=[q["id"] for q in qs], bubbles=[q["is_bubble"] for q in qs],
                         counts=[q["count"] for q in qs], next_id=opart.next_id)
    for i, q in enumerate(qs):
        p.q[i].sum, p.q[i].sumsq, p.q[i].density, p.q[i].sse = q["sum"], q["sumsq"], q["density"], q["sse"]
    return p


def to_oracle_partition(O, gpart):
    qs = gpart.queues()
    p = O.make_partition([(q["min_len"], q["max_len"]) for q in qs], means=[q["mean"] for q in qs],
                         ids=[q["id"] for q in qs], bubbles=[q["is_bubble"] for q in qs])
    p.next_id = gpart.next_id
    return p


def _close(a, b, rel=REL):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.abs(a - b) <= rel * np.maximum(np.abs(a), np.abs(b)) + 1e-30


class Report:
    def __init__(self):
        self.near_ties = 0
        self.checked_queues = 0


# Session totals (near-tie counts are reported, not silently
# tolerated): every compare_selection adds to these; conftest prints them.
SESSION = {"calls": 0, "queues": 0, "near_ties": 0, "max_per_call": 0, "unbounded_calls": 0, "unbounded_ties": 0}
# Bound per call: swapped ids are allowed only at the K-th boundary between keys
# whose fp64 scores differ by <= 1e-5 relative; more than this many in one call
# means a systematic error, not rounding.
NEAR_TIE_BOUND = 8


def compare_selection(gpu: dict, ref: dict, phi: np.ndarray, arrival: np.ndarray, mode: int, K: int,
                      base: int = 0, report: Report | None = None, near_tie_bound: int | None = NEAR_TIE_BOUND):
    """gpu: dict of numpy arrays (rows = positions); ref: oracle tick/score_select result;
    phi: oracle fp64 Φ per local request (for tie-aware checks)."""
    rep = report or Report()
    nq = ref["nq"]
    assert gpu["n_queues"] == nq, (gpu["n_queues"], nq)
    np.testing.assert_array_equal(gpu["count"][:nq], ref["count"][:nq], err_msg="counts")
    np.testing.assert_array_equal(gpu["head_id"][:nq], ref["head_id"][:nq], err_msg="head ids (FIFO key, exact)")
    ne = ref["count"][:nq] > 0
    assert _close(gpu["head_score"][:nq][ne], ref["head_score"][:nq][ne]).all(), "head_score"
    assert _close(gpu["max_score"][:nq][ne], ref["max_score"][:nq][ne]).all(), "max_score"
    for p in range(nq):
        g = gpu["topk_id"][p]
        o = ref["topk_id"][p][:K]
        m = int(min(K, ref["count"][p]))
        assert (g[m:] == -1).all() and (o[m:] == -1).all(), f"padding q{p}"
        g, o = g[:m], o[:m]
        rep.checked_queues += 1
        if m == 0:
            continue
        gl = g - base
        assert ((gl >= 0) & (gl < len(phi))).all(), f"ids out of range q{p}"
        # scores: fp32 GPU vs fp64 oracle for the same ids
        assert _close(gpu["topk_score"][p][:m], phi[gl]).all(), f"topk scores q{p}"
        if mode == 1:
            np.testing.assert_array_equal(g, o, err_msg=f"FIFO ids q{p}")
            continue
        if np.array_equal(g, o):
            continue
        # SCORE: allow swaps only among near-ties (oracle fp64 Φ within 1e-5 relative)
        sg, so = set(g.tolist()), set(o.tolist())
        boundary = phi[o[-1] - base]
        for x in sg ^ so:
            assert _close(phi[x - base], boundary), f"q{p}: id {x} differs beyond near-tie"
            rep.near_ties += 1
        pg = phi[gl]
        for a, b in zip(pg[:-1], pg[1:]):
            assert a >= b or _close(a, b), f"q{p}: GPU order violates Φ beyond near-tie"
        rep.near_ties += int((g != o).sum())
    # primary: exact unless the top two head scores are within tolerance
    hs = np.where(ne, ref["head_score"][:nq], -np.inf)
    if ne.any():
        best = hs.max()
        cands = [p for p in range(nq) if ne[p] and _close(hs[p], best)]
        if len(cands) == 1:
            assert gpu["primary"] == ref["primary"], (gpu["primary"], ref["primary"])
        else:
            assert gpu["primary"] in cands
    else:
        assert gpu["primary"] == -1
    SESSION["calls"] += 1
    SESSION["queues"] += rep.checked_queues
    if near_tie_bound is None:      # reported apart (long-prompt regime: ties are the norm, each still checked)
        SESSION["unbounded_calls"] += 1
        SESSION["unbounded_ties"] += rep.near_ties
    else:
        SESSION["near_ties"] += rep.near_ties
        SESSION["max_per_call"] = max(SESSION["max_per_call"], rep.near_ties)
    if near_tie_bound is not None:
        assert rep.near_ties <= near_tie_bound, f"{rep.near_ties} near-tie swaps in one selection (> {near_tie_bound})"
    return rep


def gpu_result(out) -> dict:
    """Outputs (torch) -> numpy dict with summary fields."""
    d = {k: getattr(out, k).cpu().numpy() for k in ("topk_id", "topk_score", "count", "head_id", "head_score",
                                                   "max_score")}
    d.update(out.summary)
    return d
