#!/usr/bin/env python
"""bench.py -- keys sorted/s of LearnedSort 2.0 on B200 (BASELINE.json metric).

Default (N=1): BASELINE config 2's first distribution, 200M fp64 Normal(0,1)
keys resident in HBM, sorted in place by ls_sort (sample + fit + two
partition rounds + in-bucket sort, all timed). N>1 (torchrun): BASELINE config
5, 1B fp64 keys per rank (50/50 Uniform[0,1e9) and Zipf(1.0) over 1e7 ranks,
seed 1000+rank), global sort with ls_sort_multi (range split + NCCL all-to-all
+ local sort).

Timing: W warm-up steps, then K timed steps between a barrier +
cuda.synchronize on both sides; every step is timed with CUDA events on the
launching stream around the sort call only (the pristine input is restored by
an untimed device copy before each step; the 1.6 GB input is larger than the
126 MB L2, so no flush is needed). Max over ranks. Prints one JSON line.

--impl reference times the CPU oracle (oracle/, single-threaded) as the
reference arm on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "keys sorted/sec (fp64/uint64) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "keys/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def wait_first(self, timeout=5.0):
        """Block until nvidia-smi has produced its first sample (it takes a
        few hundred ms to start), so the timed region is actually sampled."""
        t0 = time.monotonic()
        while self.proc and not self.lines and time.monotonic() - t0 < timeout:
            time.sleep(0.01)

    def mark(self, name):
        setattr(self, name, time.monotonic())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        t0, t1 = getattr(self, "t_start", None), getattr(self, "t_end", None)
        inside = [ln for t, ln in self.lines if t0 is None or (t0 <= t <= t1 + 0.05)]
        for ln in inside or [ln for _, ln in self.lines[-3:]]:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def phase_bytes(phase: str, n: int, st: dict) -> float:
    """Algorithmic HBM bytes of one launch of a phase, 8-byte keys.
    count1 also stores each key's 2-byte b1, which scatter1 reads back."""
    h0 = st["h0_keys"]
    if phase == "count0":
        return 8.0 * n
    if phase == "scatter0":
        return 16.0 * n
    if phase == "count1":
        return 10.0 * (n - h0) + 8.0 * h0
    if phase == "scatter1":
        return 18.0 * (n - h0) + 8.0 * h0
    if phase == "bucketsort":
        return 16.0 * st["small_keys"] + 8.0 * (st["h1_keys"])
    if phase == "big":
        return 40.0 * st["big_keys"]
    if phase == "fit":
        return 32.0 * (n / 100.0)
    return 0.0


def design_bytes(n: int, st: dict) -> float:
    """The implementation's own per-phase bytes: count1 stores
    each key's 2-byte b1, which scatter1 reads back (68 B/key on smooth inputs)."""
    return sum(phase_bytes(p, n, st) for p in ("fit", "count0", "scatter0", "count1", "scatter1",
                                                "bucketsort", "big"))


def class_bytes(n: int, st: dict) -> dict:
    """SURVEY §8(d) algorithmic bytes per key class (8-byte keys), the
    roofline numerator: U (key in a non-homogeneous level-0 bucket and a SMALL
    sub-bucket) 56 = count0 r8 + round 0 r+w 16 + round 1 r+w 16 + in-bucket
    sort r+w 16; H1 (homogeneous sub-bucket, also the single-key ones) 40;
    H0 (homogeneous level-0 bucket) 24 = count0 8 + round-0 read 8 + fill
    write 8; BIG 56 + 16 per MSD radix pass, counted here with one pass (72,
    SURVEY App. A). Plus the fit's sample gather (one 32-B sector per sampled
    key, < 1 B/key)."""
    h0, h1, big, small = st["h0_keys"], st["h1_keys"], st["big_keys"], st["small_keys"]
    single = max(0, n - h0 - h1 - big - small)
    b = 56.0 * small + 40.0 * (h1 + single) + 24.0 * h0 + 72.0 * big + 32.0 * (n / 100.0)
    return {"bytes": b, "bytes_per_key": b / n,
            "keys": {"U": small, "H1": h1 + single, "H0": h0, "BIG": big}}


def traffic_from_profiles(phase: str, n: int):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    e = d.get(phase)
    if not e or e.get("n") != n:
        return None
    return e.get("dram_bytes_per_launch")


def _ord_signed(t):
    """The total order of the keys (R12) as a signed int64 view (on device)."""
    import torch
    u = t.view(torch.int64)
    if t.dtype == torch.float64:  # totalOrder: flip the magnitude bits of negatives
        return torch.where(u < 0, u ^ torch.iinfo(torch.int64).max, u)
    return u ^ torch.iinfo(torch.int64).min  # unsigned order as signed


def is_sorted_dev(t) -> bool:
    o = _ord_signed(t)
    return bool((o[1:] >= o[:-1]).all().item())


def dup_ratio_dev(t) -> float:
    """1 - distinct/n of a sorted key array (SPEC's duplicate_ratio, bit equality)."""
    import torch
    u = t.view(torch.int64)
    n = u.numel()
    return 1.0 - (1 + int((u[1:] != u[:-1]).sum().item())) / n if n else 0.0


def multiset_hash(t):
    """(xor, sum) of splitmix64 over the 64-bit key patterns (order-free)."""
    import torch
    def c(x):
        return x - (1 << 64) if x >= (1 << 63) else x

    def lsr(z, k):
        return (z >> k) & ((1 << (64 - k)) - 1)
    z = t.view(torch.int64) + c(0x9E3779B97F4A7C15)
    z = (z ^ lsr(z, 30)) * c(0xBF58476D1CE4E5B9)
    z = (z ^ lsr(z, 27)) * c(0x94D049BB133111EB)
    z = z ^ lsr(z, 31)
    total = int(z.sum().item())
    while z.numel() > 1:
        if z.numel() & 1:
            z = torch.cat([z, z.new_zeros(1)])
        z = z[0::2] ^ z[1::2]
    return (int(z.item()) if z.numel() else 0, total)


def ncu_step_traffic(n: int):
    """Sum over the step's kernels of ncu dram bytes per launch (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    vals = [e.get("dram_bytes_per_launch") for e in d.values() if isinstance(e, dict) and e.get("n") == n]
    return sum(v for v in vals if v) or None


CONFIG_SET = ("c2_lognormal", "c2_exponential", "c2_mixgauss", "c3_zipf", "c3_rootdups", "c3_twodups",
              "c4_telemetry", "ref_uniform01", "ref_uniform_u64")


def time_configs(ls, keys, pristine, ws, cfg, stream, args, head) -> dict:
    """BASELINE configs 2-4 (and the uniform references of the duplicate
    budget) at 200M keys, on the bench's own buffers: 2 warm-up + `reps`
    timed ls_sort calls each (median), sorted + multiset checked, dup ratio
    and SURVEY §8(d) class bytes per config. Budget ratios = time / the
    uniform time of the same key type (u64: ref_uniform_u64; f64:
    ref_uniform01)."""
    import numpy as np
    import torch

    import datagen
    peak, _ = load_peaks()
    n = keys.numel()
    raw_p, raw_k = pristine.view(torch.int64), keys.view(torch.int64)
    out = {}
    reps = 5
    for wl in CONFIG_SET:
        dist_name, seed = datagen.WORKLOADS[wl]
        plan = datagen.Plan(dist_name, n, seed)
        tdt = torch.float64 if plan.dtype == np.float64 else torch.uint64
        p_ = raw_p.view(tdt)
        k_ = raw_k.view(tdt)
        plan.device(p_)
        torch.cuda.synchronize()
        ms, st = [], None
        for i in range(2 + reps):
            k_.copy_(p_)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st = ls.ls_sort(k_, cfg=cfg, ws=ws, stream=stream)
            e1.record(stream)
            e1.synchronize()
            if i >= 2:
                ms.append(e0.elapsed_time(e1))
        med = statistics.median(ms)
        cb = class_bytes(n, st)
        out[wl] = {"dtype": "f64" if tdt == torch.float64 else "u64", "ms": med, "min_ms": min(ms),
                   "keys_per_s": n / (med / 1e3), "dup_ratio": dup_ratio_dev(k_),
                   "sorted_ok": is_sorted_dev(k_), "multiset_ok": multiset_hash(k_) == multiset_hash(p_),
                   "bytes_per_key": cb["bytes_per_key"],
                   "roofline_frac": cb["bytes"] / (med / 1e3) / 1e9 / peak,
                   "phase_ms": {k: round(v, 4) for k, v in st["phase_ms"].items()},
                   "class_keys": cb["keys"]}
    out[head["config"]["workload"]] = {"dtype": head["dtype"], "ms": head["ms_per_step"],
                                       "keys_per_s": head["value"], "dup_ratio": head["dup_ratio"]}
    budget = {}
    for wl, r in out.items():
        ref = out.get("ref_uniform_u64" if r["dtype"] == "u64" else "ref_uniform01")
        if ref and wl.startswith(("c3", "c4")):
            budget[wl] = r["ms"] / ref["ms"]
    return {"results": out, "dup_budget_vs_uniform": budget, "dup_budget_limit": 1.5,
            "reps": reps, "note": "median of 5 timed ls_sort calls after 2 warm-ups, same buffers"}


# ----------------------------------------------------------------- ours ----

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import datagen
    import paper_2107_03290_b200 as ls

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()

    multi = world > 1 or args.force_multi
    wl = args.workload or ("c5_mix" if multi else "c2_normal")
    dist_name, seed = datagen.WORKLOADS[wl]
    if wl == "c5_mix":
        seed = 1000 + rank
    n = args.n or (1_000_000_000 if multi else 200_000_000)
    plan = datagen.Plan(dist_name, n, seed)
    tdt = torch.float64 if plan.dtype == np.float64 else torch.uint64
    pristine = torch.empty(n, dtype=tdt, device=dev)
    plan.device(pristine)
    keys = torch.empty_like(pristine)
    cfg = ls.config(flags=ls.LS_FLAG_PHASE_TIMING |
                    (ls.LS_FLAG_PEER_SCATTER if multi and not args.no_peer_scatter else 0))
    dt = ls.dtype_code(pristine)
    if multi:
        comm = ls.Comm.from_torch_distributed() if world > 1 else ls.Comm(0, 1, ls.Comm.unique_id())
        out_cap = int(n * 1.25) + 1_000_000
        out = torch.empty(out_cap, dtype=tdt, device=dev)
        ws = torch.empty(ls.multi_workspace_bytes(n, out_cap, world, dt, cfg), dtype=torch.uint8,
                         device=dev)
    else:
        ws = ls.workspace(n, dt, cfg, dev)
    torch.cuda.synchronize()

    def one_step():
        keys.copy_(pristine)  # untimed restore
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n_out = n
        if multi:
            n_out, st = ls.ls_sort_multi(comm, keys, out, cfg=cfg, ws=ws, stream=stream)
        else:
            st = ls.ls_sort(keys, cfg=cfg, ws=ws, stream=stream)
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1), st, n_out

    for _ in range(args.warmup):
        one_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times, stats = [], []
    with ClockSampler(local) as clk:
        clk.wait_first()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark("t_start")
        for _ in range(args.steps):
            ms, st, n_out = one_step()
            times.append(ms)
            stats.append(st)
        torch.cuda.synchronize()
        clk.mark("t_end")
        if world > 1:
            dist.barrier()
    total_ms = sum(times)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    keys_total = n * world * args.steps
    value = keys_total / (total_ms / 1e3)

    # per-phase device times (CUDA events recorded by libls on `stream`)
    st0 = stats[-1]
    phase_ms = {p: statistics.mean(s["phase_ms"][p] for s in stats) for p in ls.PHASES}
    n_local = st0["n"]
    dom = max((p for p in ls.PHASES if p != "fit"), key=lambda p: phase_ms[p])
    peak, peak_src = load_peaks()
    b = phase_bytes(dom, n_local, st0)
    achieved = b / (phase_ms[dom] / 1e3) / 1e9
    step_ms = total_ms / args.steps
    dbytes = design_bytes(n_local, st0)

    # correctness guard on the last step (on device): output non-decreasing and
    # the same multiset as the input (xor and sum of a 64-bit mix of every key)
    res = (out[: n_out] if multi else keys)
    sorted_ok = is_sorted_dev(res)
    multiset_ok = None if multi else multiset_hash(res) == multiset_hash(pristine)
    dup_ratio = None if multi else dup_ratio_dev(res)
    cb = class_bytes(n_local, st0)
    ncu_step = ncu_step_traffic(n_local)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if dt == ls.LS_F64 else "u64",
        "data": "synthetic (device Philox4x32-10 generator, datagen/)",
        "config": {"workload": wl, "distribution": dist_name, "seed": seed, "n_per_gpu": n,
                   "n_total": n * world, "l2": "inputs (8n bytes) larger than the 126 MB L2; "
                   "pristine input restored by an untimed D2D copy before each step",
                   "timed": "ls_sort_multi (split + all-to-all + local sort)" if multi else
                   "ls_sort: sample + fit + count0 + scatter0 + count1 + scatter1 + classify + "
                   "bucketsort + big path", "parallelism": f"range split x{world}" if multi else "1 GPU"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic_from_profiles(dom, n_local),
                     "algorithmic_bytes_per_launch": b, "avg_launch_ms": phase_ms[dom],
                     "peak_source": peak_src},
        # the whole step against SURVEY §8(d)'s roofline: class-weighted
        # algorithmic bytes (56 / 40 / 24 / 72 B per key) / peak
        "hbm_roofline_step": {"algorithmic_bytes": cb["bytes"], "bytes_per_key": cb["bytes_per_key"],
                              "class_keys": cb["keys"],
                              "achieved_gbs": cb["bytes"] / (step_ms / 1e3) / 1e9,
                              "frac": cb["bytes"] / (step_ms / 1e3) / 1e9 / peak,
                              "frac_8tbs": cb["bytes"] / (step_ms / 1e3) / 1e9 / 8000.0,
                              "roofline_ms": cb["bytes"] / peak / 1e6,
                              "impl_design_bytes_per_key": dbytes / n_local,
                              "ncu_dram_bytes_per_key": (ncu_step / n_local) if ncu_step else None},
        "phase_ms": phase_ms,
        "class_keys": {k: st0[k] for k in ("h0_keys", "h1_keys", "small_keys", "big_keys",
                                           "big_subbuckets", "max_group")},
        "dup_ratio": dup_ratio,
        "sorted_ok": sorted_ok,
        "multiset_ok": multiset_ok,
        "gpu_launches": int(sum(s["kernel_launches"] for s in stats)),
        "clocks": clk.summary(),
    }
    if not sorted_ok or multiset_ok is False:
        line["value"] = None
        line["error"] = "output check failed (sortedness or multiset hash)"
    if multi:
        line["n_out_rank0"] = n_out
        # per-rank device times (median over the timed steps) and the exchange:
        # keys each rank sent to other ranks cross NVLink once (8 B each); the
        # north_star roofline adds that NVLink term to the HBM one
        med_ms = float(np.median(times)) if times else 0.0
        remote = int(stats[-1].get("remote_keys", 0)) if stats else 0
        if world > 1:
            allv = [None] * world
            dist.all_gather_object(allv, (med_ms, remote, int(stats[-1].get("peer_scatter", 0))))
        else:
            allv = [(med_ms, remote, int(stats[-1].get("peer_scatter", 0)) if stats else 0)]
        nv_bytes = max(v[1] for v in allv) * 8
        nv_peak = 900.0  # GB/s per direction per B200 (NVLink 5, nominal)
        line["per_rank_ms"] = [round(v[0], 4) for v in allv]
        line["peer_scatter"] = [v[2] for v in allv]
        line["nvlink"] = {"bytes_per_rank_max": nv_bytes, "peak_gbs": nv_peak,
                          "peak_source": "nominal NVLink 5 per direction (no measured figure)",
                          "roofline_ms": nv_bytes / (nv_peak * 1e6),
                          "achieved_gbs": (nv_bytes / 1e6 / max(v[0] for v in allv)) if allv and max(v[0] for v in allv) > 0 else None}

    # e2e: the same metric through the C ABI with HOST buffers -- ls_sort_host:
    # H2D of the pinned input, the sort, D2H of the sorted keys, all inside the
    # timed region (one job at a time: PCIe-bound)
    if not multi and not args.no_e2e:
        host = torch.empty(n, dtype=tdt, pin_memory=True)
        host_pristine = pristine.cpu()
        e2e_ms = []
        for i in range(max(1, min(args.steps, 3)) + 1):
            host.copy_(host_pristine)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ls.ls_sort_host(host, keys, cfg=cfg, ws=ws, stream=stream)
            e1.record(stream)
            e1.synchronize()
            if i > 0:
                e2e_ms.append(e0.elapsed_time(e1))
        line["e2e"] = {"value": n / (statistics.mean(e2e_ms) / 1e3), "unit": UNIT,
                       "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                       "ms_per_step": statistics.mean(e2e_ms), "api": "ls_sort_host (C ABI, host buffers)",
                       "jobs_in_flight": 1}
        if args.e2e_jobs > 1:  # context: a service with several independent sorts in flight
            try:
                line["e2e_pipelined"] = e2e_pipelined(host_pristine, n, tdt, cfg, args.e2e_jobs,
                                                      max(2, min(args.steps, 4)))
            except Exception as e:
                line["e2e_pipelined"] = {"unavailable": str(e)[:200]}
        del host, host_pristine

    # the other BASELINE configs (2-4) and the uniform references of the
    # duplicate budget (north_star: high-duplicate inputs within 1.5x of
    # uniform-input time), each timed the same way on the same buffers
    if not multi and not args.no_configs and n == 200_000_000:
        line["configs"] = time_configs(ls, keys, pristine, ws, cfg, stream, args, line)
    # e2e (multi-GPU): host shard -> device (pinned, H2D inside the timed region),
    # ls_sort_multi, this rank's sorted slice -> host; max over ranks
    if multi and not args.no_e2e:
        try:
            host_in = torch.empty(n, dtype=tdt, pin_memory=True)
            host_in.copy_(pristine.cpu())
            host_out = torch.empty(out.numel(), dtype=tdt, pin_memory=True)
            e2e_ms = []
            for i in range(max(1, min(args.steps, 3)) + 1):
                if world > 1:
                    dist.barrier()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                keys.copy_(host_in, non_blocking=True)
                n_out2, _ = ls.ls_sort_multi(comm, keys, out, cfg=cfg, ws=ws, stream=stream)
                host_out[:n_out2].copy_(out[:n_out2], non_blocking=True)
                e1.record(stream)
                e1.synchronize()
                if i > 0:
                    e2e_ms.append(e0.elapsed_time(e1))
            t = sum(e2e_ms)
            if world > 1:
                tt = torch.tensor([t], device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t = float(tt.item())
            ms = t / len(e2e_ms)
            line["e2e"] = {"value": n * world / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                           "d2h_bytes_per_step": 8 * n_out, "ms_per_step": ms,
                           "api": "ls_sort_multi (torch pinned copies around it)"}
        except RuntimeError as e:  # pinned host memory unavailable
            line["e2e"] = {"value": None, "unit": UNIT, "unavailable": str(e)[:200]}

    # CPU baseline: the oracle as it stands, rank 0 at N=1, bounded sample
    if not multi and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(plan, args.cpu_sample, args.std_sample)

    if rank == 0:
        print(json.dumps(line), flush=True)
    if multi:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(plan, count: int, std_count: int) -> dict:
    """The oracle as it stands, single-threaded and pinned to one host core
    (the paper's sequential setting), on a bounded prefix of the same
    device-generated bytes; beside it, as context, std::sort(≺)
    on the same core and __gnu_parallel::sort(≺) on every core."""
    import oracle
    count = min(count, plan.n)
    h = plan_host_prefix(plan, count)
    allowed = sorted(os.sched_getaffinity(0))
    core = allowed[-1]
    os.sched_setaffinity(0, {core})
    try:
        t0 = time.perf_counter()
        oracle.sort(h)
        dt = time.perf_counter() - t0
        hs = h[: min(std_count, count)]
        t0 = time.perf_counter()
        oracle.std_sort(hs)
        dts = time.perf_counter() - t0
        ls1 = ls1_context(oracle, h[:LS1_KEYS], plan.dist)
    finally:
        os.sched_setaffinity(0, set(allowed))
    t0 = time.perf_counter()
    _, threads = oracle.parallel_sort(h)
    dtp = time.perf_counter() - t0
    return {"value": count / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"first {count} keys of the {plan.dist} workload (same device-generated "
                      f"bytes), oracle/ls2_oracle.c single-threaded, {dt:.1f} s",
            "pinned_core": core, "host_cpu": host_cpu(), "nproc": os.cpu_count(),
            "lscpu": lscpu(),
            "std_sort_1core": {"value": len(hs) / dts, "unit": UNIT, "cores": 1, "keys": len(hs),
                               "s": dts},
            "parallel_sort": {"value": count / dtp, "unit": UNIT, "cores": threads, "keys": count,
                              "s": dtp, "impl": "__gnu_parallel::sort"},
            "ls1_vs_ls2": ls1}


LS1_KEYS = 10_000_000


def ls1_context(oracle, head, dist):
    """the LearnedSort 1.0 oracle variant (spill bucket +
    exception table, oracle/ls1_oracle.c) against the LS 2.0 oracle on the
    same core and the same keys -- the host-side counterpart of the paper's
    LS 2.0 / LS 1.0 ratios (1.60x low-duplicate, >= 1.6x TwoDups, 4.78x
    high-duplicate average: P:27). Context only."""
    import datagen
    out = {"keys": LS1_KEYS, "paper": {"low_dup": 1.60, "twodups_min": 1.6, "high_dup_avg": 4.78}}
    for name, keys in ((dist, head), ("twodups", datagen.generate_host("twodups", LS1_KEYS, 1)),
                       ("zipf", datagen.generate_host("zipf", LS1_KEYS, 1))):
        t0 = time.perf_counter()
        _, st = oracle.ls1_sort(keys)
        t1 = time.perf_counter()
        oracle.sort(keys)
        t2 = time.perf_counter()
        out[name] = {"ls1_s": round(t1 - t0, 3), "ls2_s": round(t2 - t1, 3),
                     "ls2_over_ls1": round((t1 - t0) / (t2 - t1), 3),
                     "ls1_spill_keys": st["spill_keys"], "ls1_exception_keys": st["exception_keys"]}
    return out


def lscpu():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        keep = ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)",
                "CPU max MHz", "L3 cache")
        return {k.strip(): v.strip() for k, v in (ln.split(":", 1) for ln in out.splitlines() if ":" in ln)
                if k.strip() in keep}
    except Exception:
        return None


def plan_host_prefix(plan, count):
    """Device-generate the first `count` keys and copy them to the host."""
    import numpy as np
    import torch
    tdt = torch.float64 if plan.dtype == np.float64 else torch.uint64
    t = torch.empty(count, dtype=tdt, device="cuda")
    plan.device(t)
    torch.cuda.synchronize()
    a = t.view(torch.int64).cpu().numpy().view(np.uint64)
    return a.view(np.float64) if plan.dtype == np.float64 else a


def host_cpu():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical cores)"
    except OSError:
        pass
    return None


# ------------------------------------------------------------ reference ----

def run_reference(args):
    """The base contract's reference arm is, for this tier, the oracle."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    import datagen
    import oracle
    world = int(os.environ.get("WORLD_SIZE", "1"))
    wl = args.workload or ("c5_mix" if world > 1 else "c2_normal")
    dist_name, seed = datagen.WORKLOADS[wl]
    if wl == "c5_mix":
        seed = 1000
    n = args.n or (1_000_000_000 if world > 1 else 200_000_000)
    count = min(args.ref_sample, n)
    plan = datagen.Plan(dist_name, n, seed)
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:
        have_gpu = False
    h = plan_host_prefix(plan, count) if have_gpu else plan.host(0, count)
    for _ in range(args.warmup):
        oracle.sort(h)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.sort(h)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = count * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if plan.dtype == np.float64 else "u64", "data": "synthetic",
        "config": {"workload": wl, "distribution": dist_name, "seed": seed, "n_per_gpu": n,
                   "sample_per_step": count},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"first {count} keys of the {wl} workload per step",
                         "host_cpu": host_cpu()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def e2e_pipelined(host_pristine, n, tdt, cfg, jobs, steps):
    """End-to-end throughput with `jobs` independent sorts in flight, the way a
    service sorting a stream of batches runs: every job-step copies its input
    from pinned host memory (H2D), sorts it with ls_sort, and copies the sorted
    keys back to pinned host memory (D2H), all on the job's own stream; the
    H2D of one job overlaps the D2H of another (PCIe is full duplex). Timed
    with CUDA events from the first H2D to the last D2H."""
    import torch

    import paper_2107_03290_b200 as ls
    dev = torch.device("cuda")
    host_in = host_pristine if host_pristine.is_pinned() else host_pristine.pin_memory()
    streams = [torch.cuda.Stream() for _ in range(jobs)]
    bufs = [torch.empty(n, dtype=tdt, device=dev) for _ in range(jobs)]
    wss = [ls.workspace(n, ls.dtype_code(bufs[0])) for _ in range(jobs)]
    outs = [torch.empty(n, dtype=tdt, pin_memory=True) for _ in range(jobs)]

    def job(j, k_steps, ev_end):
        with torch.cuda.stream(streams[j]):
            for _ in range(k_steps):
                bufs[j].copy_(host_in, non_blocking=True)
                ls.ls_sort(bufs[j], cfg=cfg, ws=wss[j], stream=streams[j])
                outs[j].copy_(bufs[j], non_blocking=True)
            if ev_end is not None:
                ev_end.record(streams[j])
            streams[j].synchronize()

    def run(k_steps, timed):
        start = torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(jobs)]
        torch.cuda.synchronize()
        start.record(torch.cuda.current_stream())
        for s_ in streams:
            s_.wait_event(start)
        ts = [threading.Thread(target=job, args=(j, k_steps, ends[j] if timed else None))
              for j in range(jobs)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        torch.cuda.synchronize()
        return max(start.elapsed_time(e) for e in ends) if timed else None

    run(1, False)  # warm-up: allocations, first-call setup on every stream
    ms = run(steps, True)
    def prefix_ok(o):
        t = o[:100_001]
        if t.dtype == torch.float64:
            return bool((t.diff() >= 0).all())
        u = t.view(torch.int64) ^ torch.iinfo(torch.int64).min  # u64 order as signed
        return bool((u.diff() >= 0).all())

    ok = all(prefix_ok(o) for o in outs)
    del bufs, wss
    torch.cuda.empty_cache()
    total = jobs * steps
    return {"value": n * total / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
            "d2h_bytes_per_step": 8 * n, "ms_per_step": ms / total, "jobs_in_flight": jobs,
            "job_steps": total, "api": "ls_sort + pinned-host copies on the job's stream",
            "prefix_sorted_ok": ok}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default=None, help="a key of datagen.WORKLOADS")
    ap.add_argument("--n", type=int, default=0, help="keys per GPU (default: the config's)")
    ap.add_argument("--cpu-sample", type=int, default=100_000_000)
    ap.add_argument("--ref-sample", type=int, default=10_000_000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-jobs", type=int, default=2,
                    help="independent sorts in flight for the e2e throughput (1: one at a time)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--std-sample", type=int, default=30_000_000,
                    help="keys for the 1-core std::sort context baseline")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the other 200M configs (dup budget) in the N=1 line")
    ap.add_argument("--no-peer-scatter", action="store_true",
                    help="multi-GPU: NCCL all-to-all instead of the fused peer-store scatter (SURVEY f1)")
    ap.add_argument("--force-multi", action="store_true",
                    help="run the ls_sort_multi path (config 5) even at world size 1")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup < 3 is below the contract minimum", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
