"""LearnedSort 2.0 (arXiv 2107.03290) hot path on B200 -- Python binding of libls.so.

Thin layer over the C ABI in include/ls.h: every step of the sort runs in the
CUDA kernels of libls.so; this module only marshals torch tensors (device
memory, streams) into the C calls. It raises ImportError when libls.so is
missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

from . import _lib
from ._lib import (LS_E_CAPACITY, LS_E_CUDA, LS_E_INTERNAL, LS_E_INVALID, LS_E_NAN, LS_E_NCCL,
                   LS_E_WORKSPACE, LS_F64, LS_FLAG_FUSED_ROUND1, LS_FLAG_PEER_SCATTER, LS_FLAG_PHASE_TIMING, LS_OK,
                   LS_U64, PHASES, Config,
                   Dumps, Leaf, Model, Stats, Tagged)

lib = _lib.load()

__all__ = [
    "lib", "LSError", "config", "dtype_code", "workspace_bytes", "workspace", "ls_train_rmi",
    "ls_sort", "ls_sort_with_model", "ls_sort_host", "ls_bucket_ids", "Comm", "ls_sort_multi",
    "multi_workspace_bytes", "multi_splitters", "multi_plan", "multi_dest", "multi_sample",
    "multi_route", "Config", "Model",
    "Stats", "Dumps", "Tagged", "Leaf", "PHASES", "LS_F64", "LS_U64", "LS_OK", "LS_E_NAN",
    "LS_E_INVALID", "LS_E_WORKSPACE", "LS_E_CAPACITY", "LS_E_CUDA", "LS_E_NCCL", "LS_E_INTERNAL",
    "LS_FLAG_PHASE_TIMING", "LS_FLAG_FUSED_ROUND1", "LS_FLAG_PEER_SCATTER", "multi_route_peer",
]


class LSError(RuntimeError):
    def __init__(self, status: int, where: str):
        name = lib.ls_status_string(status).decode()
        detail = lib.ls_last_error().decode()
        super().__init__(f"{where}: {name} ({detail})")
        self.status = status


def _check(status: int, where: str) -> None:
    if status != LS_OK:
        raise LSError(status, where)


def config(fanout: int = 1000, leaf_count: int = 1000, sample_stride: int = 100,
           big_threshold: int = 4096, flags: int = 0) -> Config:
    c = Config()
    lib.ls_config_default(C.byref(c))
    c.fanout, c.leaf_count, c.sample_stride = fanout, leaf_count, sample_stride
    c.big_threshold, c.flags = big_threshold, flags
    return c


def dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float64:
        return LS_F64
    if t.dtype == torch.uint64:
        return LS_U64
    raise TypeError(f"keys must be torch.float64 or torch.uint64, got {t.dtype}")


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def workspace_bytes(n: int, dtype: int = LS_F64, cfg: Config | None = None) -> int:
    out = C.c_size_t()
    _check(lib.ls_workspace_bytes(n, dtype, C.byref(cfg or config()), C.byref(out)),
           "ls_workspace_bytes")
    return out.value


def workspace(n: int, dtype: int = LS_F64, cfg: Config | None = None, device="cuda"):
    import torch
    return torch.empty(max(workspace_bytes(n, dtype, cfg), 256), dtype=torch.uint8, device=device)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def ls_train_rmi(sample, cfg: Config | None = None, ws=None, stream=None) -> Model:
    """Fit F_A on a device sample tensor (north_star (1))."""
    cfg = cfg or config()
    dt = dtype_code(sample)
    ws = ws if ws is not None else workspace(sample.numel(), dt, cfg, sample.device)
    m = Model()
    _check(lib.ls_train_rmi(_ptr(sample), sample.numel(), dt, C.byref(cfg), C.byref(m),
                            _ptr(ws), ws.numel(), _stream(stream)), "ls_train_rmi")
    return m


def ls_sort(keys, cfg: Config | None = None, ws=None, stream=None, dumps: Dumps | None = None,
            model: Model | None = None) -> dict:
    """Sort a contiguous 1-D float64/uint64 CUDA tensor in place. Returns stats."""
    cfg = cfg or config()
    dt = dtype_code(keys)
    assert keys.is_cuda and keys.is_contiguous()
    ws = ws if ws is not None else workspace(keys.numel(), dt, cfg, keys.device)
    st = Stats()
    if model is None:
        rc = lib.ls_sort(_ptr(keys), keys.numel(), dt, C.byref(cfg), _ptr(ws), ws.numel(),
                         _stream(stream), C.byref(st), C.byref(dumps) if dumps else None)
    else:
        rc = lib.ls_sort_with_model(_ptr(keys), keys.numel(), dt, C.byref(cfg), C.byref(model),
                                    _ptr(ws), ws.numel(), _stream(stream), C.byref(st),
                                    C.byref(dumps) if dumps else None)
    _check(rc, "ls_sort")
    return st.as_dict()


def ls_sort_with_model(keys, model: Model, **kw) -> dict:
    return ls_sort(keys, model=model, **kw)


def ls_sort_host(host_keys, dev_buf, cfg: Config | None = None, ws=None, stream=None) -> dict:
    """End-to-end: host tensor (pinned) -> device -> sort -> host, one C call."""
    cfg = cfg or config()
    dt = dtype_code(host_keys)
    n = host_keys.numel()
    ws = ws if ws is not None else workspace(n, dt, cfg, dev_buf.device)
    st = Stats()
    _check(lib.ls_sort_host(C.c_void_p(host_keys.data_ptr()), n, dt, C.byref(cfg), _ptr(dev_buf),
                            _ptr(ws), ws.numel(), _stream(stream), C.byref(st)), "ls_sort_host")
    return st.as_dict()


def ls_bucket_ids(keys, model: Model, cfg: Config | None = None, ws=None, stream=None,
                  want=("p", "b0", "b1", "pos", "hist0", "hist1")) -> dict:
    """Per-key p / b0 / b1 / pos and raw histograms for a given model (parity hook)."""
    import torch
    cfg = cfg or config()
    dt = dtype_code(keys)
    n, f, dev = keys.numel(), cfg.fanout, keys.device
    ws = ws if ws is not None else workspace(n, dt, cfg, dev)
    out = {}
    if "p" in want:
        out["p"] = torch.empty(n, dtype=torch.float64, device=dev)
    for k in ("b0", "b1", "pos"):
        if k in want:
            out[k] = torch.empty(n, dtype=torch.int32, device=dev)
    if "hist0" in want:
        out["hist0"] = torch.empty(f, dtype=torch.int64, device=dev)
    if "hist1" in want:
        out["hist1"] = torch.empty(f * f, dtype=torch.int64, device=dev)
    g = out.get
    _check(lib.ls_bucket_ids(_ptr(keys), n, dt, C.byref(cfg), C.byref(model), _ptr(g("p")),
                             _ptr(g("b0")), _ptr(g("b1")), _ptr(g("pos")), _ptr(g("hist0")),
                             _ptr(g("hist1")), _ptr(ws), ws.numel(), _stream(stream)),
           "ls_bucket_ids")
    return out


# --------------------------------------------------------------- multi-GPU --

class Comm:
    """NCCL communicator owned by libls (ls_comm). Bootstrap via torch.distributed."""

    def __init__(self, rank: int, world: int, uid: bytes):
        self.rank, self.world = rank, world
        h = C.c_void_p()
        buf = (C.c_uint8 * _lib.LS_UNIQUE_ID_BYTES).from_buffer_copy(uid)
        _check(lib.ls_comm_init(buf, rank, world, C.byref(h)), "ls_comm_init")
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * _lib.LS_UNIQUE_ID_BYTES)()
        _check(lib.ls_comm_unique_id(buf), "ls_comm_unique_id")
        return bytes(buf)

    @classmethod
    def from_torch_distributed(cls):
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(rank, world, obj[0])

    def close(self):
        if self.handle:
            lib.ls_comm_destroy(self.handle)
            self.handle = None


def multi_workspace_bytes(n_in: int, out_cap: int, world: int, dtype: int = LS_F64,
                          cfg: Config | None = None) -> int:
    out = C.c_size_t()
    _check(lib.ls_multi_workspace_bytes(n_in, out_cap, world, dtype, C.byref(cfg or config()),
                                        C.byref(out)), "ls_multi_workspace_bytes")
    return out.value


def ls_sort_multi(comm: Comm, keys_in, out, cfg: Config | None = None, ws=None,
                  stream=None) -> tuple[int, dict]:
    """SPMD global sort: returns (n_out, stats); out[:n_out] is this rank's slice."""
    import torch
    cfg = cfg or config()
    dt = dtype_code(keys_in)
    if ws is None:
        ws = torch.empty(multi_workspace_bytes(keys_in.numel(), out.numel(), comm.world, dt, cfg),
                         dtype=torch.uint8, device=keys_in.device)
    n_out = C.c_uint64()
    st = Stats()
    _check(lib.ls_sort_multi(comm.handle, _ptr(keys_in), keys_in.numel(), _ptr(out), out.numel(),
                             C.byref(n_out), dt, C.byref(cfg), _ptr(ws), ws.numel(), _stream(stream),
                             C.byref(st)), "ls_sort_multi")
    return n_out.value, st.as_dict()


def multi_splitters(entries, world: int):
    """entries: numpy structured array (ord u8, rank u4, pad u4, index u8); sorted in place."""
    import numpy as np
    spl = np.zeros(max(world - 1, 1), dtype=entries.dtype)
    _check(lib.ls_multi_splitters(entries.ctypes.data, len(entries), world, spl.ctypes.data),
           "ls_multi_splitters")
    return spl[: world - 1]


def multi_plan(counts, world: int, rank: int):
    import numpy as np
    counts = np.ascontiguousarray(counts, dtype=np.uint64)
    sd = np.zeros(world, np.uint64)
    rc_ = np.zeros(world, np.uint64)
    rd = np.zeros(world, np.uint64)
    n_out = C.c_uint64()
    _check(lib.ls_multi_plan(counts.ctypes.data, world, rank, sd.ctypes.data, rc_.ctypes.data,
                             rd.ctypes.data, C.byref(n_out)), "ls_multi_plan")
    return sd, rc_, rd, n_out.value


TAGGED_DTYPE = [("ord", "<u8"), ("rank", "<u4"), ("pad", "<u4"), ("index", "<u8")]


def multi_sample(keys, rank: int, stream=None):
    """The LS_MULTI_SAMPLE tagged split-sample entries of one rank's shard
    (step 1 of ls_sort_multi), as a numpy structured array."""
    import numpy as np
    import torch
    d = torch.empty(_lib.LS_MULTI_SAMPLE * 24, dtype=torch.uint8, device=keys.device)
    _check(lib.ls_multi_sample(_ptr(keys), keys.numel(), rank, dtype_code(keys), _ptr(d),
                               _stream(stream)), "ls_multi_sample")
    return d.cpu().numpy().view(np.dtype(TAGGED_DTYPE)).copy()


def multi_route(keys, rank: int, world: int, splitters, send, ws=None, stream=None):
    """Steps 3 + 5 of ls_sort_multi for one rank without a communicator: returns
    the destination counts; send[:n] holds the shard grouped by destination."""
    import numpy as np
    import torch
    dt = dtype_code(keys)
    if ws is None:
        ws = torch.empty(multi_workspace_bytes(keys.numel(), 0, world, dt), dtype=torch.uint8,
                         device=keys.device)
    spl = np.ascontiguousarray(splitters)
    counts = np.zeros(world, np.uint64)
    _check(lib.ls_multi_route(_ptr(keys), keys.numel(), rank, world,
                              spl.ctypes.data if len(spl) else None, dt, _ptr(send),
                              counts.ctypes.data, _ptr(ws), ws.numel(), _stream(stream)),
           "ls_multi_route")
    return counts


def multi_route_peer(keys, rank: int, world: int, splitters, dsts, offsets, ws=None, stream=None):
    """SURVEY f1's fused destination scatter for one rank without a
    communicator: destination p's keys are stored into the device tensor
    dsts[p] from element offsets[p] on; returns the destination counts."""
    import numpy as np
    import torch
    dt = dtype_code(keys)
    if ws is None:
        ws = torch.empty(multi_workspace_bytes(keys.numel(), 0, world, dt), dtype=torch.uint8,
                         device=keys.device)
    spl = np.ascontiguousarray(splitters)
    ptrs = (C.c_void_p * world)(*[_ptr(d) for d in dsts])
    offs = np.ascontiguousarray(offsets, dtype=np.uint64)
    counts = np.zeros(world, np.uint64)
    _check(lib.ls_multi_route_peer(_ptr(keys), keys.numel(), rank, world,
                                   spl.ctypes.data if len(spl) else None, dt, ptrs,
                                   offs.ctypes.data, counts.ctypes.data, _ptr(ws), ws.numel(),
                                   _stream(stream)), "ls_multi_route_peer")
    return counts


def multi_dest(splitters, world: int, ord_: int, rank: int, index: int) -> int:
    return lib.ls_multi_dest(splitters.ctypes.data if len(splitters) else None, world, ord_, rank,
                             index)
