"""Fill BASELINE.md §3 (results table) from one evidence run:
gpurun_out/configs.jsonl (one bench line per workload), gpurun_out/bench.json
(the headline line with cpu_baseline). Prints the markdown table; with
--write replaces the table in BASELINE.md."""
import json
import sys

ROWS = [  # (config, label, workload, dtype, parity at full size / at 1e6-1e7)
    ("1", "Uniform[0,1)", "c1_uniform01", "fp64", "1e6/1e7 element-wise"),
    ("2", "Normal(0,1)", "c2_normal", "fp64", "200M element-wise + S_B/S'_B/H0/H1"),
    ("2", "LogNormal(0,0.5)", "c2_lognormal", "fp64", "200M element-wise + S_B/S'_B/H0/H1"),
    ("2", "Exponential(λ=2)", "c2_exponential", "fp64", "200M element-wise + S_B/S'_B/H0/H1"),
    ("2", "5-Gaussian mix", "c2_mixgauss", "fp64", "200M element-wise + S_B/S'_B/H0/H1"),
    ("3", "Zipf(0.75), 1M values", "c3_zipf", "u64", "200M element-wise + S_B/S'_B/H0/H1"),
    ("3", "RootDups", "c3_rootdups", "u64", "200M element-wise + S_B/S'_B/H0/H1"),
    ("3", "TwoDups", "c3_twodups", "u64", "200M element-wise + S_B/S'_B/H0/H1"),
    ("4", "telemetry levels + ID clusters", "c4_telemetry", "u64", "200M element-wise + S_B/S'_B/H0/H1"),
    ("ref", "Uniform[0,1)", "ref_uniform01", "fp64", "200M element-wise + S_B/S'_B/H0/H1"),
    ("ref", "uniform u64", "ref_uniform_u64", "u64", "200M element-wise + S_B/S'_B/H0/H1"),
]


def main():
    lines = [json.loads(l) for l in open("gpurun_out/configs.jsonl") if l.strip().startswith("{")]
    by = {d["config"]["workload"]: d for d in lines if "config" in d and "workload" in d["config"]}
    head = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
    cb = head.get("cpu_baseline", {})
    l12 = cb.get("ls1_vs_ls2", {})
    keys = l12.get("keys", 0)
    orc = {"c2_normal": cb.get("value")}
    for wl, k in (("c3_twodups", "twodups"), ("c3_zipf", "zipf")):
        if k in l12 and keys:
            orc[wl] = keys / l12[k]["ls2_s"]
    std1 = cb.get("std_sort_1core", {}).get("value")
    out = ["| Config | Distribution | dtype | n (total) | GPUs | dup ratio (measured) | GPU keys/s | ms/step | "
           "% HBM roofline (8 TB/s) | % (measured peak) | Oracle keys/s (1 core) | std::sort keys/s (1 core) | "
           "Parity (GPU tests) |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    try:  # config 1 (1M keys) from the graph-latency run: same buffers, graph replay, median of 30
        gl = [json.loads(l) for l in open("gpurun_out/graph_latency.jsonl") if l.strip()]
        g1 = next(x for x in gl if x["n"] == 1_000_000 and x["graph"])
        out.append(f"| 1 | Uniform[0,1) | fp64 | 1M | 1 | — | {g1['gkeys_per_s']:.2f} G | {g1['ms_median']:.3f} | "
                   f"— (launch-latency bound) | — | — | — | 1e6 element-wise |")
    except (OSError, StopIteration):
        pass
    for cfg, label, wl, dt, par in ROWS:
        d = by.get(wl)
        if d is None or wl == "c1_uniform01":
            continue
        r = d.get("hbm_roofline_step", {})
        o = orc.get(wl)
        n = d["config"]["n_total"]
        out.append(f"| {cfg} | {label} | {dt} | {n / 1e6:.0f}M | 1 | {d.get('dup_ratio', 0):.4f} | "
                   f"{d['value'] / 1e9:.1f} G | {d['ms_per_step']:.3f} | {100 * r.get('frac_8tbs', 0):.1f} % | "
                   f"{100 * r.get('frac', 0):.1f} % | {f'{o / 1e6:.1f} M' if o else '—'} | "
                   f"{f'{std1 / 1e6:.1f} M' if (std1 and wl == 'c2_normal') else '—'} | {par} |")
    fm = [d for d in lines if d.get("config", {}).get("workload", "").startswith("c5")]
    for d in fm:
        out.append(f"| 5 | Uniform[0,1e9) + Zipf(1.0), one-rank `ls_sort_multi` | fp64 | "
                   f"{d['config']['n_total'] / 1e9:.0f}B | 1 | — | {d['value'] / 1e9:.1f} G | {d['ms_per_step']:.2f} | — | — | — | — | "
                   f"routing on 2..8 virtual ranks; 1-rank NCCL |")
    out.append("| 5 | Uniform[0,1e9) + Zipf(1.0) | fp64 | 2B / 4B / 8B | 2 / 4 / 8 | | not measured (1-GPU pool) | | | | | | |")
    table = "\n".join(out)
    print(table)
    if "--write" in sys.argv:
        s = open("BASELINE.md").read()
        a = s.index("## 3. Results")
        b = s.find("\n## ", a + 5)
        hdr = ("## 3. Results (B200, filled from the round's evidence run: `profiles/"
               + (sys.argv[sys.argv.index("--tag") + 1] if "--tag" in sys.argv else "rNN") + "_configs.jsonl`)\n\n")
        s = s[:a] + hdr + table + "\n" + (s[b:] if b > 0 else "")
        open("BASELINE.md", "w").write(s)


if __name__ == "__main__":
    main()
