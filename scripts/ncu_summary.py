"""Summarise ncu outputs into profiles/: the launch list (per-kernel device
time and share of the step) and one `--set full` capture (per-kernel DRAM
traffic, throughput, instructions). Also writes profiles/ncu_traffic.json,
which bench.py reads for roofline.traffic."""
import collections
import csv
import json
import subprocess
import sys

PHASE_OF = {"k_count0": "count0", "k_scatter0": "scatter0", "k_scatter0r": "scatter0", "k_count1": "count1",
            "k_scatter1": "scatter1", "k_warpsort": "bucketsort", "k_bucketsort": "bucketsort", "k_ctasort": "bucketsort",
            "k_big": "big"}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    agg = collections.defaultdict(list)
    for r in rows:
        if len(r) == len(hdr) and r[0] != "ID":
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0].replace("void ", "")
                v = float(d["Metric Value"].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
                agg[name].append(v)  # usecond
    ours = {k: v for k, v in agg.items() if k.startswith("ls::")}
    tot = sum(sum(v) for v in ours.values())
    lines = ["| kernel | launches | avg us | share of libls time |", "|---|---|---|---|"]
    for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")
    others = {k: v for k, v in agg.items() if not k.startswith("ls::")}
    lines.append("")
    lines.append("Not libls (bench harness: input generator, torch sortedness check): " +
                 ", ".join(f"{k.split('<')[0]} x{len(v)}" for k, v in others.items()))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def full(rep, out, n):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = ["| kernel | " + " | ".join(m.split("__")[1] if "__" in m else m for m in METRICS) + " |",
             "|---" * (len(METRICS) + 1) + "|"]
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        vals = []
        for m in METRICS:
            i = hdr.index(m) if m in hdr else None
            vals.append(f"{r[i]} {units[i]}".strip() if i is not None else "-")
        lines.append(f"| {name} | " + " | ".join(vals) + " |")
        base = name.split("<")[0]
        ph = PHASE_OF.get(base)
        if ph:
            def val(m):
                i = hdr.index(m)
                x = float(r[i].replace(",", ""))
                u = units[i]
                return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            e = traffic.setdefault(ph, {"n": n, "dram_bytes_per_launch": 0.0, "kernel": ""})
            e["dram_bytes_per_launch"] += val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
            e["kernel"] = (e["kernel"] + " + " if e["kernel"] else "") + name
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)


if __name__ == "__main__":
    tag = sys.argv[1]
    launches("gpurun_out/launches.csv", f"profiles/{tag}_launches.md")
    full("gpurun_out/prof_full.ncu-rep", f"profiles/{tag}_ncu_full.md", int(sys.argv[2]) if len(sys.argv) > 2 else 200_000_000)
