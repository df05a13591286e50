"""Maximum sizes: n above 2^31 and just below the C ABI's limit (n < 2^32,
include/ls.h): sorts device-generated keys through ls_sort and checks, in
chunks, that the output is non-decreasing under the key order and is the same
multiset as the input (two wrapping sums over a 64-bit mix of every word), and that
n = 2^32 is rejected with LS_E_INVALID. One JSON line per point."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2107_03290_b200 as ls  # noqa: E402

CH = 1 << 28


def words_hash(t):
    u = t.view(torch.int64)
    s, s2 = 0, 0
    for i in range(0, u.numel(), CH):
        c = u[i:i + CH]
        m = c * -7046029254386353131  # (odd multiplier, wrapping: a bijection on words)
        m = m ^ (m >> 29)
        s = (s + int(m.sum().item())) & ((1 << 64) - 1)
        s2 = (s2 + int((m * (m | 1)).sum().item())) & ((1 << 64) - 1)
    return s, s2


def sorted_ok(t, f64):
    u = t.view(torch.int64)
    last = None
    for i in range(0, u.numel(), CH):
        c = u[i:i + CH]
        o = torch.where(c < 0, c ^ torch.iinfo(torch.int64).max, c) if f64 else c ^ torch.iinfo(torch.int64).min
        if not bool((o[1:] >= o[:-1]).all().item()):
            return False
        if last is not None and int(o[0].item()) < last:
            return False
        last = int(o[-1].item())
    return True


def run(dist, n):
    plan = datagen.Plan(dist, n, 0)
    f64 = plan.dtype == np.float64
    src = torch.empty(n, dtype=torch.float64 if f64 else torch.uint64, device="cuda")
    plan.device(src)
    h0 = words_hash(src)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = ls.ls_sort(src)
    e1.record()
    e1.synchronize()
    out = {"dist": dist, "n": n, "ms": e0.elapsed_time(e1), "sorted_ok": sorted_ok(src, f64),
           "multiset_ok": words_hash(src) == h0, "small_keys": st["small_keys"], "h1_keys": st["h1_keys"],
           "big_keys": st["big_keys"]}
    del src
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    for dist, n in (("normal", 2_500_000_000), ("twodups", 2_500_000_000), ("normal", 4_294_967_295)):
        print(json.dumps(run(dist, n)), flush=True)
    try:
        b = ls.workspace_bytes(1 << 32, 0)
        print(json.dumps({"n": 1 << 32, "rejected": False, "workspace_bytes": b}))
    except ls.LSError as e:
        print(json.dumps({"n": 1 << 32, "rejected": True, "status": e.status}))
