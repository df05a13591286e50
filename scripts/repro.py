"""Sort one synthetic input through the C ABI and compare with the oracle (debug aid)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen, oracle as O
import paper_2107_03290_b200 as ls
ap = argparse.ArgumentParser()
ap.add_argument("--dist", default="twodups"); ap.add_argument("--n", type=int, default=3_000_000)
ap.add_argument("--seed", type=int, default=29); ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--check", action="store_true")
a = ap.parse_args()
plan = datagen.Plan(a.dist, a.n, a.seed)
tdt = torch.float64 if plan.dtype == np.float64 else torch.uint64
src = torch.empty(a.n, dtype=tdt, device="cuda"); plan.device(src)
for r in range(a.reps):
    t = src.clone(); st = ls.ls_sort(t); torch.cuda.synchronize()
    print("rep", r, "ok", st["big_subbuckets"], st["max_group"])
if a.check:
    h = src.view(torch.int64).cpu().numpy().view(np.uint64)
    h = h.view(np.float64) if plan.dtype == np.float64 else h
    got = t.view(torch.int64).cpu().numpy().view(np.uint64)
    print("equal:", np.array_equal(got, O.sort(h)[0].view(np.uint64)))
