"""Large-size randomised stress run of ls_sort on the GPU (30M..400M keys,
duplicate-heavy generators included): each output is compared with torch.sort
of the same keys under the same total order (ord), on the device."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen, paper_2107_03290_b200 as ls
rng = np.random.default_rng(5)
DISTS = ["normal", "zipf", "twodups", "telemetry", "rootdups", "cfg5mix", "lognormal", "uniform_u64"]
fails = 0
t_end = time.time() + 300
runs = 0
while time.time() < t_end:
    dist = DISTS[rng.integers(len(DISTS))]
    n = int(rng.integers(30_000_000, 400_000_000))
    seed = int(rng.integers(1 << 30))
    kw = {}
    if rng.random() < 0.3: kw["big_threshold"] = int(rng.choice([64, 256, 1024]))
    plan = datagen.Plan(dist, n, seed)
    tdt = torch.float64 if plan.dtype == np.float64 else torch.uint64
    t = torch.empty(n, dtype=tdt, device="cuda"); plan.device(t)
    def key(x):
        u = x.view(torch.int64)
        if x.dtype == torch.float64:
            return torch.where(u < 0, u ^ torch.iinfo(torch.int64).max, u)
        return u ^ torch.iinfo(torch.int64).min
    ref = torch.sort(key(t)).values
    try:
        ls.ls_sort(t, cfg=ls.config(**kw))
        ok = bool(torch.equal(key(t), ref))
    except Exception as e:
        ok = False; print("ERROR", dist, n, seed, kw, e, flush=True)
    runs += 1
    if not ok:
        fails += 1; print("FAIL", dist, n, seed, kw, flush=True)
    del t, ref; torch.cuda.empty_cache()
print(f"bigstress: {runs} runs, {fails} failures")
