"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper around oracle/liboracle.so.

The plain CPU oracle of LearnedSort 2.0 (arXiv 2107.03290); see
oracle/ls2_oracle.c for the step-by-step citations. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module. It never imports the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

F64, U64 = 0, 1
OK, E_INVALID, E_NAN, E_INTERNAL = 0, 1, 2, 7
MAX_LEAVES = 4096


class Leaf(C.Structure):
    _fields_ = [("a", C.c_double), ("c", C.c_double), ("b", C.c_double),
                ("lo", C.c_double), ("hi", C.c_double)]


class Model(C.Structure):
    _fields_ = [("leaf_count", C.c_uint32), ("degenerate", C.c_uint32),
                ("n_sample", C.c_uint64), ("xmin", C.c_double), ("xmax", C.c_double),
                ("root_scale", C.c_double), ("leaf", Leaf * MAX_LEAVES)]

    def leaves(self) -> np.ndarray:
        """[L, 5] array of (a, c, b, lo, hi)."""
        arr = np.ctypeslib.as_array(self.leaf).view(np.float64).reshape(MAX_LEAVES, 5)
        return arr[: self.leaf_count].copy()


class Frag(C.Structure):
    _fields_ = [("bucket", C.c_uint64), ("size", C.c_uint64)]


class Config(C.Structure):
    _fields_ = [("fanout", C.c_uint32), ("leaf_count", C.c_uint32),
                ("sample_stride", C.c_uint32), ("frag_capacity", C.c_uint32)]


class Dumps(C.Structure):
    _fields_ = [("p", C.c_void_p), ("b0", C.c_void_p), ("b1", C.c_void_p),
                ("pos", C.c_void_p), ("S_B", C.c_void_p), ("S_B1", C.c_void_p),
                ("hist1_raw", C.c_void_p), ("H0", C.c_void_p), ("H1", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "h0_buckets", "h0_keys", "h1_subbuckets", "h1_keys", "counting_sorts",
        "shifts", "guard_fired", "max_group", "max_subbucket")]

    def as_dict(self) -> dict:
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class LS1Config(C.Structure):
    """ls1o_config (oracle/ls1_oracle.c)."""
    _fields_ = [("fanout", C.c_uint32), ("leaf_count", C.c_uint32),
                ("sample_stride", C.c_uint32), ("slack", C.c_double), ("cap0", C.c_uint64),
                ("cap1", C.c_uint64), ("exc_min", C.c_uint64)]


class LS1Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "spill_l0", "spill_keys", "exception_values", "exception_keys", "shifts", "guard_fired")]

    def as_dict(self) -> dict:
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc (no contraction, no fast-math)."""
    srcs = [os.path.join(_HERE, f) for f in ("ls2_oracle.c", "ls1_oracle.c")]
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            [os.path.getmtime(x) for x in srcs] + [os.path.getmtime(os.path.join(_HERE, "ls2_oracle.h"))]):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-Wall", "-o", _SO] + srcs + ["-lm"])
    return _SO


_lib = None
_HS_SO = os.path.join(_HERE, "libhostsorts.so")
_hs = None


def build_host_sorts(force: bool = False) -> str:
    """std::sort(≺) and __gnu_parallel::sort(≺) (oracle/host_sorts.cpp): the
    CPU context baselines of bench.py's cpu_baseline leg."""
    src = os.path.join(_HERE, "host_sorts.cpp")
    if force or not os.path.exists(_HS_SO) or os.path.getmtime(_HS_SO) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared", "-Wall",
                               "-o", _HS_SO, src])
    return _HS_SO


def host_sorts():
    global _hs
    if _hs is None:
        build_host_sorts()
        L = C.CDLL(_HS_SO)
        L.lso_std_sort.argtypes = [C.c_void_p, C.c_uint64, C.c_int]
        L.lso_parallel_sort.argtypes = [C.c_void_p, C.c_uint64, C.c_int]
        L.lso_parallel_sort.restype = C.c_int
        _hs = L
    return _hs


def std_sort(keys: np.ndarray) -> np.ndarray:
    """std::sort with the total-order comparator, on the calling thread."""
    a = keys.copy()
    host_sorts().lso_std_sort(_u64(a).ctypes.data, len(a), dtype_code(keys))
    return a


def parallel_sort(keys: np.ndarray):
    """__gnu_parallel::sort with the same comparator; returns (sorted, threads)."""
    a = keys.copy()
    th = host_sorts().lso_parallel_sort(_u64(a).ctypes.data, len(a), dtype_code(keys))
    return a, th


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        P = C.c_void_p
        L.lso_config_default.argtypes = [C.POINTER(Config)]
        L.lso_ord.argtypes = [C.c_uint64, C.c_int]; L.lso_ord.restype = C.c_uint64
        L.lso_xd.argtypes = [C.c_uint64, C.c_int]; L.lso_xd.restype = C.c_double
        L.lso_train.argtypes = [P, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32, C.POINTER(Model)]
        L.lso_predict.argtypes = [C.POINTER(Model), C.c_uint64, C.c_int]; L.lso_predict.restype = C.c_double
        L.lso_bucket_l0.argtypes = [C.c_double, C.c_uint32]; L.lso_bucket_l0.restype = C.c_uint64
        L.lso_bucket_l1.argtypes = [C.c_double, C.c_uint32, C.c_uint64]; L.lso_bucket_l1.restype = C.c_uint64
        L.lso_cs_pos.argtypes = [C.c_double, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64]
        L.lso_cs_pos.restype = C.c_uint64
        L.lso_partition.argtypes = [P, C.c_uint64, C.POINTER(Model), C.c_int, C.c_int, C.c_uint64,
                                    C.c_uint32, C.c_uint32, P, P]
        L.lso_partition.restype = C.c_uint64
        L.lso_defragment.argtypes = [P, C.c_uint64, C.c_uint32, P, P, C.c_uint64, P]
        L.lso_is_homogeneous.argtypes = [P, C.c_uint64, C.c_int]
        L.lso_counting_sort.argtypes = [P, C.c_uint64, C.POINTER(Model), C.c_int, C.c_uint64,
                                        C.c_uint64, C.c_uint32, C.c_uint64, P, P]
        L.lso_counting_sort.restype = C.c_uint64
        L.lso_insertion_sort.argtypes = [P, C.c_uint64, C.c_int, C.c_uint64, C.POINTER(C.c_int)]
        L.lso_insertion_sort.restype = C.c_uint64
        L.lso_sort.argtypes = [P, C.c_uint64, C.c_int, C.POINTER(Config), C.POINTER(Model),
                               C.POINTER(Model), C.POINTER(Dumps), C.POINTER(Stats)]
        L.lso_reference_sort.argtypes = [P, C.c_uint64, C.c_int]
        L.ls1o_config_default.argtypes = [C.POINTER(LS1Config)]
        L.ls1o_sort.argtypes = [P, C.c_uint64, C.c_int, C.POINTER(LS1Config), C.POINTER(LS1Stats)]
        _lib = L
    return _lib


# ----------------------------------------------------------------- helpers --

def _u64(keys: np.ndarray) -> np.ndarray:
    keys = np.ascontiguousarray(keys)
    assert keys.dtype.itemsize == 8
    return keys.view(np.uint64)


def dtype_code(keys: np.ndarray) -> int:
    return F64 if keys.dtype == np.float64 else U64


def config(fanout=1000, leaf_count=1000, sample_stride=100, frag_capacity=100) -> Config:
    return Config(fanout, leaf_count, sample_stride, frag_capacity)


def ord_key(keys: np.ndarray) -> np.ndarray:
    """Vectorised ord (same definition as lso_ord, for test-side checks)."""
    u = _u64(keys)
    if keys.dtype == np.float64:
        neg = (u >> np.uint64(63)).astype(bool)
        return np.where(neg, ~u, u | np.uint64(1 << 63))
    return u.copy()


def train(keys: np.ndarray, stride=100, leaf_count=1000) -> Model:
    u = _u64(keys)
    m = Model()
    rc = lib().lso_train(u.ctypes.data, len(u), dtype_code(keys), stride, leaf_count, C.byref(m))
    if rc != OK:
        raise RuntimeError(f"lso_train rc={rc}")
    return m


def predict(model: Model, keys: np.ndarray) -> np.ndarray:
    u = _u64(keys)
    d = dtype_code(keys)
    L = lib()
    return np.array([L.lso_predict(C.byref(model), int(x), d) for x in u], dtype=np.float64)


def sort(keys: np.ndarray, cfg: Config | None = None, model: Model | None = None,
         dumps: bool | str = False):
    """Run Alg. 2 on a copy. Returns (sorted, model, stats, dumps-dict|None).
    dumps=True: every dump; dumps="tables": only the per-bucket tables (S_B,
    S'_B, hist1_raw, H0, H1), no per-key arrays (full-size runs)."""
    a = keys.copy()
    u = _u64(a)
    n = len(u)
    cfg = cfg or config()
    f = cfg.fanout
    mo = Model()
    st = Stats()
    dd = None
    dp = None
    if dumps:
        dd = dict(S_B=np.zeros(f, np.uint64), S_B1=np.zeros(f * f, np.uint64),
                  hist1_raw=np.zeros(f * f, np.uint64), H0=np.zeros(f, np.uint8),
                  H1=np.zeros(f * f, np.uint8))
        if dumps != "tables":
            dd.update(p=np.zeros(n, np.float64), b0=np.zeros(n, np.uint32),
                      b1=np.zeros(n, np.uint32), pos=np.zeros(n, np.uint32))
        dp = Dumps(*[dd[k].ctypes.data if k in dd else None
                     for k in ("p", "b0", "b1", "pos", "S_B", "S_B1", "hist1_raw", "H0", "H1")])
    rc = lib().lso_sort(u.ctypes.data, n, dtype_code(keys), C.byref(cfg),
                        C.byref(model) if model is not None else None, C.byref(mo),
                        C.byref(dp) if dp is not None else None, C.byref(st))
    if rc != OK:
        raise OracleError(rc)
    return a, mo, st.as_dict(), dd


class OracleError(RuntimeError):
    def __init__(self, rc):
        super().__init__(f"oracle status {rc}")
        self.rc = rc


def reference_sort(keys: np.ndarray) -> np.ndarray:
    a = keys.copy()
    lib().lso_reference_sort(_u64(a).ctypes.data, len(a), dtype_code(keys))
    return a


def ls1_config(fanout=1000, leaf_count=1000, sample_stride=100, slack=1.1, cap0=0, cap1=0,
               exc_min=0) -> LS1Config:
    return LS1Config(fanout, leaf_count, sample_stride, slack, cap0, cap1, exc_min)


def ls1_sort(keys: np.ndarray, cfg: LS1Config | None = None):
    """LearnedSort 1.0 (oracle variant) on a copy.
    Returns (sorted, stats-dict)."""
    a = keys.copy()
    u = _u64(a)
    st = LS1Stats()
    rc = lib().ls1o_sort(u.ctypes.data, len(u), dtype_code(keys), C.byref(cfg or ls1_config()),
                         C.byref(st))
    if rc != OK:
        raise OracleError(rc)
    return a, st.as_dict()
