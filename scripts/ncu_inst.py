"""Per-source-line warp instructions / active lanes / stall samples for one kernel."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
nkeys = float(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None
hdr = None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        inst = int(r[hdr.index("Instructions Executed")] or 0)
        th = int(r[hdr.index("Thread Instructions Executed")] or 0)
        smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    a = agg.setdefault((cur, int(r[0])), [0, 0, 0, r[1][:80]])
    a[0] += inst
    a[1] += th
    a[2] += smp
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[2] for v in agg.values()) or 1
print(f"warp inst {tot}" + (f"  per key {tot / nkeys:.2f}" if nkeys else ""))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:>11d} {100 * v[0] / tot:5.1f}% lanes {v[1] / max(v[0], 1):4.1f} stall {100 * v[2] / ts:5.1f}%  {k[0]}:{k[1]:<4d} {v[3]}")
