"""Level-0 bucket size distribution (hist0) of a synthetic input: how many
buckets / keys would fit a cluster-resident round 1 of a given capacity."""
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
ap.add_argument("--n", type=int, default=200_000_000)
a = ap.parse_args()
plan = datagen.Plan(a.dist, a.n, 0)
tdt = torch.float64 if plan.dtype == np.float64 else torch.uint64
keys = torch.empty(a.n, dtype=tdt, device="cuda")
plan.device(keys)
sample = keys[::100].contiguous()
model = ls.ls_train_rmi(sample)
out = ls.ls_bucket_ids(keys, model, want=("hist0",))
h = out["hist0"].cpu().numpy()
print(a.dist, a.n, "buckets", len(h), "mean", h.mean(), "max", h.max(), "p50/p90/p99",
      np.percentile(h, [50, 90, 99]))
for cap in (150_000, 200_000, 208_000, 250_000, 300_000, 400_000, 420_000):
    fit = h <= cap
    print(f"cap {cap}: buckets {fit.sum()} keys {h[fit].sum() / h.sum():.3f}")
