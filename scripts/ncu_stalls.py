"""Stall breakdown (warp-cycles per issued instruction by reason) and pipe
utilisation for each kernel in an ncu report."""
import csv
import subprocess
import sys

rep = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    name = d.get("Kernel Name", "")
    if flt not in name:
        continue
    print(name[:60], d.get("gpu__time_duration.sum", ""))
    st = []
    for k, x in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(x), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("  stalls/issue:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:9]))
    pp = []
    for k, x in d.items():
        if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active"):
            try:
                if float(x) > 3:
                    pp.append((float(x), k[len("sm__inst_executed_pipe_"):-len(".avg.pct_of_peak_sustained_active")]))
            except ValueError:
                pass
    print("  pipes %:", ", ".join(f"{n} {x:.0f}" for x, n in sorted(pp, reverse=True)))
    for k in ("sm__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_op_red.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"):
        if k in d:
            print("  ", k, d[k])
