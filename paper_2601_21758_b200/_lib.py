"""ctypes declarations of the libewsjf C ABI (include/ewsjf.h).  Marshalling only.

The CUDA library is required: importing this module on a machine where
``libewsjf.so`` is missing raises immediately (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libewsjf_check.so" if os.environ.get("EWSJF_CHECKED") == "1" else "libewsjf.so")

MAX_QUEUES = 256
HIST_BINS = 1 << 20
MAX_K = 256

OK, INVALID_ARG, DOMAIN, EMPTY, CAPACITY, CUDA_ERR, UNSUPPORTED, NCCL_ERR = range(8)
NCCL_ID_BYTES = 128
SELECT_SCORE, SELECT_FIFO = 0, 1
MIN_U, MAX_U = 0, 1


class PartitionParams(C.Structure):
    _fields_ = [("alpha", C.c_double), ("min_width", C.c_int32), ("max_queues", C.c_int32),
                ("epsilon", C.c_double), ("coarse_k", C.c_int32), ("merge_rule", C.c_int32),
                ("gap_rule", C.c_int32), ("kmeans_k", C.c_int32)]


class Queue(C.Structure):
    _fields_ = [("id", C.c_int32), ("index", C.c_int32), ("min_len", C.c_int32), ("max_len", C.c_int32),
                ("count", C.c_int64), ("sum", C.c_int64), ("sumsq", C.c_int64),
                ("mean", C.c_double), ("density", C.c_double), ("sse", C.c_double),
                ("is_bubble", C.c_int32), ("empty_count", C.c_int32)]


class Partition(C.Structure):
    _fields_ = [("n", C.c_int32), ("next_id", C.c_int32), ("version", C.c_uint64), ("q", Queue * MAX_QUEUES)]

    def queues(self) -> list[dict]:
        return [{f: getattr(self.q[i], f) for f, _ in Queue._fields_} for i in range(self.n)]


class PartitionStats(C.Structure):
    _fields_ = [("n_valid", C.c_int64), ("n_invalid", C.c_int64), ("distinct", C.c_int64),
                ("k_used", C.c_int32), ("t1", C.c_int32), ("t2", C.c_int32), ("segments", C.c_int64),
                ("depth", C.c_int32), ("merges", C.c_int64),
                ("ms_hist", C.c_float), ("ms_kmeans", C.c_float), ("ms_refine", C.c_float),
                ("ms_prune", C.c_float), ("ms_total", C.c_float)]


class Meta(C.Structure):
    _fields_ = [(f, C.c_double) for f in ("a_b", "b_b", "a_u", "b_u", "a_f", "b_f")]


class Weights(C.Structure):
    _fields_ = [("w_base", C.c_float), ("w_urg", C.c_float), ("w_fair", C.c_float)]


class CostParams(C.Structure):
    _fields_ = [("c0", C.c_float), ("c1", C.c_float), ("c2", C.c_float)]


class SelectParams(C.Structure):
    _fields_ = [("k", C.c_int32), ("mode", C.c_int32), ("now", C.c_float), ("cost", CostParams)]


class Summary(C.Structure):
    _fields_ = [("n_queues", C.c_int32), ("primary", C.c_int32), ("n_invalid", C.c_int64),
                ("n_excluded", C.c_int64), ("n_gap", C.c_int64), ("n_bubbles", C.c_int64),
                ("n_dropped", C.c_int64), ("status", C.c_int32), ("pad", C.c_int32)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "pad"}


class Timing(C.Structure):
    _fields_ = [("launches", C.c_int64), ("recorded", C.c_int64), ("tick_launches", C.c_int64),
                ("merge_launches", C.c_int64), ("partition_launches", C.c_int64), ("sweep_launches", C.c_int64),
                ("tick_ms", C.c_double), ("merge_ms", C.c_double), ("partition_ms", C.c_double),
                ("sweep_ms", C.c_double), ("candidates_inserted", C.c_int64), ("compactions", C.c_int64),
                ("batch_launches", C.c_int64), ("batch_ms", C.c_double), ("sweep_records", C.c_int64)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


class Budget(C.Structure):
    _fields_ = [("max_requests", C.c_int32), ("pad", C.c_int32), ("max_tokens", C.c_int64)]


class SelectOut(C.Structure):
    _fields_ = [("d_topk_id", C.c_void_p), ("d_topk_score", C.c_void_p), ("d_count", C.c_void_p),
                ("d_head_id", C.c_void_p), ("d_head_score", C.c_void_p), ("d_max_score", C.c_void_p),
                ("d_summary", C.c_void_p), ("h_summary", C.POINTER(Summary))]


# every symbol include/ewsjf.h declares (checked by tests/test_abi.py)
SYMBOLS = [
    "ewsjf_abi_version", "ewsjf_status_str", "ewsjf_last_error", "ewsjf_ctx_create", "ewsjf_ctx_set_stream",
    "ewsjf_ctx_destroy", "ewsjf_ctx_num_ctas", "ewsjf_partition", "ewsjf_weights_from_meta", "ewsjf_route",
    "ewsjf_score_select", "ewsjf_tick", "ewsjf_tick_host", "ewsjf_exchange_bytes", "ewsjf_tick_local",
    "ewsjf_tick_merge", "ewsjf_score_select_sweep", "ewsjf_ctx_set_timing", "ewsjf_ctx_get_timing",
    "ewsjf_ctx_get_phases", "ewsjf_batch_build", "ewsjf_prune_empty",
    "ewsjf_history_hist", "ewsjf_partition_from_hist", "ewsjf_online_adjust",
    "ewsjf_nccl_get_unique_id", "ewsjf_ctx_init_nccl", "ewsjf_ctx_attach_nccl", "ewsjf_ctx_detach_nccl",
    "ewsjf_diag_ffma_rate", "ewsjf_ctx_reserve_sweep", "ewsjf_alloc_count", "ewsjf_ctx_set_exchange_gap_cap",
]

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libewsjf.so not built at {LIB_PATH}: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P, V, I32, I64 = C.POINTER, C.c_void_p, C.c_int32, C.c_int64
    L.ewsjf_abi_version.restype = C.c_int
    L.ewsjf_status_str.restype = C.c_char_p
    L.ewsjf_status_str.argtypes = [C.c_int]
    L.ewsjf_last_error.restype = C.c_char_p
    L.ewsjf_last_error.argtypes = [V]
    L.ewsjf_ctx_create.argtypes = [C.c_int, V, I64, I64, I32, P(V)]
    L.ewsjf_ctx_set_stream.argtypes = [V, V]
    L.ewsjf_ctx_destroy.argtypes = [V]
    L.ewsjf_ctx_num_ctas.argtypes = [V]
    L.ewsjf_ctx_num_ctas.restype = I32
    L.ewsjf_ctx_set_timing.argtypes = [V, I32]
    L.ewsjf_ctx_get_timing.argtypes = [V, P(Timing)]
    L.ewsjf_ctx_get_phases.argtypes = [V, P(C.c_uint64), I32]
    L.ewsjf_partition.argtypes = [V, V, I64, P(PartitionParams), P(Partition), P(PartitionStats)]
    L.ewsjf_weights_from_meta.argtypes = [P(Meta), P(Partition), P(Weights)]
    L.ewsjf_route.argtypes = [V, V, I64, P(Partition), I32, V, P(Summary)]
    L.ewsjf_score_select.argtypes = [V, V, V, V, V, I64, P(Partition), P(Weights), P(SelectParams), P(SelectOut)]
    L.ewsjf_tick.argtypes = [V, V, V, V, I64, I64, P(Partition), I32, P(Meta), P(SelectParams), V, P(SelectOut)]
    L.ewsjf_tick_host.argtypes = [V, V, V, V, I64, I64, P(Partition), I32, P(Meta), P(SelectParams), V, V, V, V,
                                  V, V, V, P(Summary)]
    L.ewsjf_exchange_bytes.argtypes = [V, I32, I32]
    L.ewsjf_exchange_bytes.restype = I64
    L.ewsjf_tick_local.argtypes = [V, V, V, V, I64, I64, P(Partition), P(Meta), P(SelectParams), V, V]
    L.ewsjf_tick_merge.argtypes = [V, V, I32, I64, I64, V, P(Partition), I32, P(Meta), P(SelectParams),
                                   P(SelectOut)]
    L.ewsjf_score_select_sweep.argtypes = [V, V, V, V, V, I64, P(Partition), P(Meta), I32, P(SelectParams),
                                           P(SelectOut)]
    L.ewsjf_batch_build.argtypes = [V, V, I64, I64, P(SelectOut), I32, I32, P(Budget), V, V]
    L.ewsjf_prune_empty.argtypes = [P(Partition), V, I32, P(C.c_int32)]
    L.ewsjf_history_hist.argtypes = [V, V, I64, V, P(C.c_int64)]
    L.ewsjf_online_adjust.argtypes = [V, V, I64, C.c_double, P(Partition), P(C.c_int32)]
    L.ewsjf_partition_from_hist.argtypes = [V, V, I32, I64, P(PartitionParams), P(Partition), P(PartitionStats)]
    L.ewsjf_nccl_get_unique_id.argtypes = [V]
    L.ewsjf_ctx_init_nccl.argtypes = [V, V, I32, I32]
    L.ewsjf_ctx_attach_nccl.argtypes = [V, V, I32, I32]
    L.ewsjf_ctx_detach_nccl.argtypes = [V]
    L.ewsjf_diag_ffma_rate.argtypes = [V, P(C.c_double)]
    L.ewsjf_ctx_reserve_sweep.argtypes = [V, I64]
    L.ewsjf_ctx_set_exchange_gap_cap.argtypes = [V, I32]
    L.ewsjf_alloc_count.argtypes = []
    L.ewsjf_alloc_count.restype = I64
    for name in SYMBOLS:
        if name not in ("ewsjf_abi_version", "ewsjf_status_str", "ewsjf_last_error", "ewsjf_ctx_num_ctas",
                        "ewsjf_exchange_bytes", "ewsjf_alloc_count"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L
