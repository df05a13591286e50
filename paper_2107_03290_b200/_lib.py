"""ctypes declarations of libls.so (include/ls.h). Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("LS_LIBPATH") or os.path.join(_HERE, "libls.so")  # (override: A/B runs)

LS_F64, LS_U64 = 0, 1
LS_OK, LS_E_INVALID, LS_E_NAN, LS_E_WORKSPACE, LS_E_CAPACITY, LS_E_CUDA, LS_E_NCCL, LS_E_INTERNAL = range(8)
LS_MAX_FANOUT = 1024
LS_MAX_LEAVES = 1024
LS_FLAG_PHASE_TIMING = 0x1
LS_FLAG_VALIDATE_MODEL = 0x2
LS_FLAG_FUSED_ROUND1 = 0x4
LS_FLAG_PEER_SCATTER = 0x8
LS_MULTI_SAMPLE = 16384
LS_UNIQUE_ID_BYTES = 128
PHASES = ("fit", "count0", "scatter0", "count1", "scatter1", "classify", "bucketsort", "big")

# Every function include/ls.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "ls_config_default", "ls_status_string", "ls_last_error", "ls_workspace_bytes",
    "ls_train_rmi", "ls_sort", "ls_sort_with_model", "ls_sort_host", "ls_bucket_ids",
    "ls_comm_unique_id", "ls_comm_init", "ls_comm_destroy", "ls_multi_workspace_bytes",
    "ls_sort_multi", "ls_multi_splitters", "ls_multi_plan", "ls_multi_dest", "ls_multi_sample",
    "ls_multi_route", "ls_multi_route_peer",
)


class Config(C.Structure):
    _fields_ = [("fanout", C.c_uint32), ("leaf_count", C.c_uint32), ("sample_stride", C.c_uint32),
                ("fit", C.c_uint32), ("big_threshold", C.c_uint32), ("reserved", C.c_uint32),
                ("flags", C.c_uint64)]


class Leaf(C.Structure):
    _fields_ = [("a", C.c_double), ("c", C.c_double), ("b", C.c_double),
                ("lo", C.c_double), ("hi", C.c_double)]


class Model(C.Structure):
    _fields_ = [("dtype", C.c_uint32), ("leaf_count", C.c_uint32), ("n_sample", C.c_uint64),
                ("degenerate", C.c_uint32), ("reserved", C.c_uint32),
                ("xmin", C.c_double), ("xmax", C.c_double), ("root_scale", C.c_double),
                ("leaf", Leaf * LS_MAX_LEAVES)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "n", "h0_buckets", "h0_keys", "h1_subbuckets", "h1_keys", "small_subbuckets",
        "small_keys", "big_subbuckets", "big_keys", "max_group", "big_passes",
        "kernel_launches", "fused_buckets", "round0_exact", "peer_scatter", "remote_keys")] + [("phase_ms", C.c_float * len(PHASES))]

    def as_dict(self) -> dict:
        d = {n: int(getattr(self, n)) for n, _ in self._fields_[:-1]}
        d["phase_ms"] = {p: float(self.phase_ms[i]) for i, p in enumerate(PHASES)}
        return d


class Dumps(C.Structure):
    _fields_ = [("d_S_B", C.c_void_p), ("d_S_B1", C.c_void_p), ("d_H0", C.c_void_p),
                ("d_H1", C.c_void_p), ("h_model", C.POINTER(Model))]


class Tagged(C.Structure):
    _fields_ = [("ord", C.c_uint64), ("rank", C.c_uint32), ("pad", C.c_uint32), ("index", C.c_uint64)]


def load() -> C.CDLL:
    if not os.path.exists(SO_PATH):
        raise ImportError(
            f"{SO_PATH} is missing: build it with `make` (or __graft_entry__.build()). "
            "There is no fallback path.")
    L = C.CDLL(SO_PATH)
    P, U64, U32, I = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
    S = C.c_int  # ls_status
    sig = {
        "ls_config_default": (None, [C.POINTER(Config)]),
        "ls_status_string": (C.c_char_p, [S]),
        "ls_last_error": (C.c_char_p, []),
        "ls_workspace_bytes": (S, [U64, I, C.POINTER(Config), C.POINTER(C.c_size_t)]),
        "ls_train_rmi": (S, [P, U64, I, C.POINTER(Config), C.POINTER(Model), P, C.c_size_t, P]),
        "ls_sort": (S, [P, U64, I, C.POINTER(Config), P, C.c_size_t, P, C.POINTER(Stats),
                        C.POINTER(Dumps)]),
        "ls_sort_with_model": (S, [P, U64, I, C.POINTER(Config), C.POINTER(Model), P, C.c_size_t, P,
                                   C.POINTER(Stats), C.POINTER(Dumps)]),
        "ls_sort_host": (S, [P, U64, I, C.POINTER(Config), P, P, C.c_size_t, P, C.POINTER(Stats)]),
        "ls_bucket_ids": (S, [P, U64, I, C.POINTER(Config), C.POINTER(Model), P, P, P, P, P, P, P,
                              C.c_size_t, P]),
        "ls_comm_unique_id": (S, [P]),
        "ls_comm_init": (S, [P, I, I, C.POINTER(P)]),
        "ls_comm_destroy": (None, [P]),
        "ls_multi_workspace_bytes": (S, [U64, U64, I, I, C.POINTER(Config), C.POINTER(C.c_size_t)]),
        "ls_sort_multi": (S, [P, P, U64, P, U64, C.POINTER(U64), I, C.POINTER(Config), P, C.c_size_t,
                              P, C.POINTER(Stats)]),
        "ls_multi_splitters": (S, [P, U64, I, P]),
        "ls_multi_plan": (S, [P, I, I, P, P, P, C.POINTER(U64)]),
        "ls_multi_dest": (I, [P, I, U64, U32, U64]),
        "ls_multi_sample": (S, [P, U64, I, I, P, P]),
        "ls_multi_route": (S, [P, U64, I, I, P, I, P, P, P, C.c_size_t, P]),
        "ls_multi_route_peer": (S, [P, U64, I, I, P, I, P, P, P, P, C.c_size_t, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L
