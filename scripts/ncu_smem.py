"""Per CUDA source line: shared-memory wavefronts (actual / ideal) and stall
samples, from `ncu --page source --print-source cuda,sass`."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None
agg = {}
hdr = None
src_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if not r[0].isdigit():  # SASS rows: the CUDA line row already aggregates them
        continue
    try:
        wf = float(r[hdr.index("L1 Wavefronts Shared")] or 0)
        ideal = float(r[hdr.index("L1 Wavefronts Shared Ideal")] or 0)
    except (ValueError, IndexError):
        continue
    key = (cur, r[0], r[1][:70])
    a = agg.setdefault(key, [0, 0])
    a[0] += wf
    a[1] += ideal
tot = sum(v[0] for v in agg.values()) or 1
print(f"total shared wavefronts {tot:.3e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}% {v[0]:.3e} ideal {v[1]:.3e}  {k[0]}:{k[1]} {k[2]}")
