"""Summarise `ncu --page source --print-source cuda,sass --csv` per CUDA source
line: stall samples and executed warp instructions, hottest first."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
fname_filter = sys.argv[4] if len(sys.argv) > 4 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = None
cur_fn = ''
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        cur_fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    if fname_filter and fname_filter not in cur_fn:
        continue
    try:
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        inst = int(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    if samp == 0 and inst == 0:
        continue
    key = (cur_file, int(r[0]))
    a = agg.setdefault(key, [0, 0, r[1][:90]])
    a[0] += samp
    a[1] += inst
tot = sum(v[0] for v in agg.values()) or 1
print(f"total stall samples {tot}")
for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/tot:5.1f}% {i:>12d}  {f}:{ln:<5d} {src}")
