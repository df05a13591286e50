"""The paper's second workloads on B200 (Fig. 5 / Fig. 6):

  * size sweep (Fig. 5): Normal(0,1) fp64 and TwoDups u64 from 1M
    to 1B keys -- keys/s per size (the paper's "cache-size knee" is an L2
    effect here: inputs up to ~8M keys stay in the 126 MB L2);
  * Zipf skew sweep (Fig. 6): Zipf(s) u64 over V = 1M values,
    s = 0.50 .. 0.99, 200M keys -- keys/s per skew, and the ratio to
    Normal(0,1) at the same size (the paper reports LS2.0 losing only 3 % at
    s = 0.99 relative to its Normal reference);
  * Chi-square(k = 4) fp64 at 200M.

Every point sorts device-generated synthetic keys through the C ABI
(ls_sort), timed with CUDA events on the launching stream (median of K runs
after W warm-ups), checks that the output is non-decreasing, and prints one
JSON line per point."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2107_03290_b200 as ls  # noqa: E402


def run(dist, n, seed, reps, warm, **kw):
    plan = datagen.Plan(dist, n, seed, **kw)
    tdt = torch.float64 if plan.dtype == np.float64 else torch.uint64
    src = torch.empty(n, dtype=tdt, device="cuda")
    plan.device(src)
    keys = torch.empty_like(src)
    ws = ls.workspace(n, ls.dtype_code(src))
    stream = torch.cuda.current_stream()
    times = []
    for r in range(warm + reps):
        keys.copy_(src)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st = ls.ls_sort(keys, ws=ws, stream=stream)
        e1.record(stream)
        e1.synchronize()
        if r >= warm:
            times.append(e0.elapsed_time(e1))
    u = keys.view(torch.int64)
    o = torch.where(u < 0, u ^ torch.iinfo(torch.int64).max, u) if tdt == torch.float64 \
        else u ^ torch.iinfo(torch.int64).min
    ok = bool((o[1:] >= o[:-1]).all().item())
    ms = statistics.median(times)
    del src, keys, ws
    torch.cuda.empty_cache()
    return {"dist": dist, "n": n, "ms": ms, "keys_per_s": n / (ms / 1e3), "sorted_ok": ok,
            "small_keys": st["small_keys"], "h1_keys": st["h1_keys"], "big_keys": st["big_keys"],
            **{k: v for k, v in kw.items()}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--max-n", type=int, default=1_000_000_000)
    a = ap.parse_args()
    sizes = [n for n in (1_000_000, 4_000_000, 16_000_000, 64_000_000, 200_000_000, 500_000_000,
                         1_000_000_000) if n <= a.max_n]
    for dist in ("normal", "twodups"):
        for n in sizes:
            print(json.dumps({"sweep": "size", **run(dist, n, 0, a.reps, a.warmup)}), flush=True)
    ref = run("normal", 200_000_000, 0, a.reps, a.warmup)
    for s in (0.5, 0.6, 0.7, 0.75, 0.8, 0.9, 0.95, 0.99):
        r = run("zipf", 200_000_000, 1, a.reps, a.warmup, zipf_s=s, zipf_V=1_000_000)
        r["vs_normal"] = r["keys_per_s"] / ref["keys_per_s"]
        print(json.dumps({"sweep": "zipf_skew", **r}), flush=True)
    print(json.dumps({"sweep": "chisq4", **run("chisq4", 200_000_000, 0, a.reps, a.warmup)}),
          flush=True)


if __name__ == "__main__":
    main()
