"""Randomised stress run of ls_sort on the GPU: random sizes, distributions,
seeds and configurations (fan-out, big threshold, fused round 1), each output
compared bit for bit with numpy's sort under the same total order (ord). Prints
one line per failure and a summary; exit status 1 on any failure."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2107_03290_b200 as ls  # noqa: E402

DISTS = ["uniform01", "normal", "lognormal", "exponential", "mixgauss", "chisq4", "zipf", "rootdups",
         "twodups", "telemetry", "uniform_u64", "cfg5mix"]


def ord_sorted(a: np.ndarray) -> np.ndarray:
    b = a.view(np.uint64)
    if a.dtype == np.float64:
        neg = (b >> np.uint64(63)) == 1
        o = np.where(neg, ~b, b | np.uint64(1 << 63))
    else:
        o = b
    return b[np.argsort(o, kind="stable")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=240)
    ap.add_argument("--max-n", type=int, default=3_000_000)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    t_end = time.time() + a.seconds
    runs = fails = 0
    while time.time() < t_end:
        dist = DISTS[rng.integers(len(DISTS))]
        n = int(rng.choice([rng.integers(0, 3000), rng.integers(0, 300_000), rng.integers(0, a.max_n)]))
        seed = int(rng.integers(1 << 30))
        kw = {}
        if rng.random() < 0.3:
            kw["fanout"] = int(rng.choice([2, 3, 16, 100, 1000, 1024]))
        if rng.random() < 0.3:
            kw["big_threshold"] = int(rng.choice([64, 100, 512, 1024, 4096]))
        if rng.random() < 0.2:
            kw["flags"] = ls.LS_FLAG_FUSED_ROUND1
            os.environ["LS_FR_MIN"] = str(int(rng.choice([256, 4096, 65536])))
        else:
            os.environ.pop("LS_FR_MIN", None)
        if rng.random() < 0.25:  # host-made patterns: order, few values, clusters, specials
            pat = int(rng.integers(7))
            r2 = np.random.default_rng(seed)
            if pat == 0:
                h = np.sort(r2.standard_normal(n))
            elif pat == 1:
                h = np.sort(r2.standard_normal(n))[::-1].copy()
            elif pat == 2:
                h = np.full(n, r2.standard_normal())
            elif pat == 3:
                h = r2.integers(0, int(r2.integers(1, 17)), n).astype(np.uint64)
            elif pat == 4:
                h = (r2.integers(0, 4, n) * 1e6 + r2.integers(0, 1000, n) * 1e-9).astype(np.float64)
            elif pat == 5:
                sp = np.array([np.inf, -np.inf, 0.0, -0.0, 5e-324, -5e-324, 1e308, -1e308])
                h = np.where(r2.random(n) < 0.3, sp[r2.integers(0, len(sp), n)], r2.standard_normal(n))
            else:
                h = (np.uint64(1) << np.uint64(63)) + r2.integers(0, 2 ** 20, n).astype(np.uint64)
            dist = f"pattern{pat}"
            tdt = torch.float64 if h.dtype == np.float64 else torch.uint64
            t = torch.from_numpy(h.view(np.int64).copy()).cuda().view(tdt)
        else:
            try:
                plan = datagen.Plan(dist, n, seed)
            except Exception:  # (generator limits, e.g. twodups n < 2^32)
                continue
            tdt = torch.float64 if plan.dtype == np.float64 else torch.uint64
            t = torch.empty(n, dtype=tdt, device="cuda")
            if n:
                plan.device(t)
            h = t.view(torch.int64).cpu().numpy().view(np.uint64).view(plan.dtype).copy()
        try:
            ls.ls_sort(t, cfg=ls.config(**kw))
            got = t.view(torch.int64).cpu().numpy().view(np.uint64)
            ok = np.array_equal(got, ord_sorted(h))
        except Exception as e:  # noqa: BLE001
            ok = False
            print(f"ERROR {dist} n={n} seed={seed} cfg={kw}: {e}", flush=True)
        runs += 1
        if not ok:
            fails += 1
            print(f"FAIL {dist} n={n} seed={seed} cfg={kw} fr_min={os.environ.get('LS_FR_MIN')}", flush=True)
        del t
    print(f"stress: {runs} runs, {fails} failures")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
