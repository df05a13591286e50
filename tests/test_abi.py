"""The C-ABI library loads and exports every symbol include/ls.h declares (CPU)."""
import ctypes as C
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ls.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(ls_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    import paper_2107_03290_b200 as ls
    from paper_2107_03290_b200 import _lib
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(ls.lib, n), n
    assert set(names) == set(_lib.EXPORTS)


def test_host_only_entry_points():
    """Calls that never touch the GPU: config, status strings, workspace sizing,
    and argument validation (errors are returned, not raised, across the ABI)."""
    import paper_2107_03290_b200 as ls
    c = ls.config()
    assert (c.fanout, c.leaf_count, c.sample_stride) == (1000, 1000, 100)
    assert ls.lib.ls_status_string(ls.LS_E_NAN) == b"LS_E_NAN"
    n = 200_000_000
    wb = ls.workspace_bytes(n)
    # scratch B (n + n/4 + 4096 f keys: round 0's reserved bucket regions), its
    # bucket ids, task and big lists
    assert 10 * n <= wb <= 15 * n + 200 * 2 ** 20
    bad = ls.config(fanout=1)
    out = C.c_size_t()
    assert ls.lib.ls_workspace_bytes(10, 0, C.byref(bad), C.byref(out)) == ls.LS_E_INVALID
    st = ls.Stats()
    # n <= 1 is a no-op that succeeds without touching memory
    assert ls.lib.ls_sort(None, 1, 0, None, None, 0, None, C.byref(st), None) == ls.LS_OK
    assert ls.lib.ls_sort(C.c_void_p(16), 1 << 32, 0, None, C.c_void_p(16), 1 << 40, None,
                          None, None) == ls.LS_E_INVALID
    assert ls.lib.ls_sort(C.c_void_p(16), 100, 0, None, C.c_void_p(256), 1, None, None,
                          None) == ls.LS_E_WORKSPACE
    assert b"workspace" in ls.lib.ls_last_error()
    # keys at an odd 8-byte offset / an unaligned workspace: rejected before any work
    assert ls.lib.ls_sort(C.c_void_p(24), 100, 0, None, C.c_void_p(256), 1 << 40, None, None,
                          None) == ls.LS_E_INVALID
    assert b"aligned" in ls.lib.ls_last_error()
    assert ls.lib.ls_sort(C.c_void_p(16), 100, 0, None, C.c_void_p(272), 1 << 40, None, None,
                          None) == ls.LS_E_INVALID
    # ls_sort_host with n <= 1: returns before any copy is queued (nothing left
    # in flight that could land in the caller's buffer after the call)
    st.n = 99
    assert ls.lib.ls_sort_host(C.c_void_p(8), 1, 0, None, None, None, 0, None, C.byref(st)) == ls.LS_OK
    assert st.n == 1
    # multi entry points validate the config before any layout arithmetic
    # (sample_stride = 0 would divide by zero) or collective
    z = ls.config()
    z.sample_stride = 0
    assert ls.lib.ls_multi_workspace_bytes(1000, 1000, 2, 0, C.byref(z), C.byref(out)) == ls.LS_E_INVALID
    assert b"sample_stride" in ls.lib.ls_last_error()
    n_out = C.c_uint64()
    assert ls.lib.ls_sort_multi(None, None, 0, None, 0, C.byref(n_out), 0, C.byref(z), None, 0, None,
                                None) == ls.LS_E_INVALID
    # structure sizes agree with the header (offsets of the trailing members)
    assert C.sizeof(ls.Model) == 4 + 4 + 8 + 4 + 4 + 3 * 8 + 1024 * 40
    assert C.sizeof(ls.Tagged) == 24
