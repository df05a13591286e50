"""Sort one synthetic input twice (warm-up + measured) for ncu captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2107_03290_b200 as ls  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dist", default="normal")
ap.add_argument("--n", type=int, default=50_000_000)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--flags", type=lambda x: int(x, 0), default=0, help="extra LS_FLAG_* bits")
ap.add_argument("--big", type=int, default=4096, help="big_threshold of the config")
a = ap.parse_args()
plan = datagen.Plan(a.dist, a.n, a.seed)
tdt = torch.float64 if plan.dtype == np.float64 else torch.uint64
src = torch.empty(a.n, dtype=tdt, device="cuda")
plan.device(src)
keys = torch.empty_like(src)
ws = ls.workspace(a.n, ls.dtype_code(src))
for r in range(a.reps):
    keys.copy_(src)
    st = ls.ls_sort(keys, ws=ws, cfg=ls.config(flags=ls.LS_FLAG_PHASE_TIMING | a.flags, big_threshold=a.big))
    print(r, {k: round(v, 3) for k, v in st["phase_ms"].items()}, st["small_keys"], st["h1_keys"],
          st["big_keys"])
torch.cuda.synchronize()
