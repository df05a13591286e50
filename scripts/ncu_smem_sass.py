"""Per-SASS-instruction shared-memory wavefronts (actual / ideal) of one kernel
from an ncu report: where the bank conflicts are."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
c = {k: h.index(k) for k in ("Instructions Executed", "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal",
                             "Warp Stall Sampling (All Samples)")}
tot = 0
res = []
for r in rows[2:]:
    try:
        w = int(r[c["L1 Wavefronts Shared"]] or 0)
        wi = int(r[c["L1 Wavefronts Shared Ideal"]] or 0)
        n = int(r[c["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    tot += w
    if w:
        res.append((w, wi, n, r[1].strip()))
print(f"total shared wavefronts {tot}")
for w, wi, n, s in sorted(res, reverse=True)[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{w / 1e6:8.2f}M ideal {wi / 1e6:7.2f}M  per-inst {w / max(n, 1):5.2f}  {s[:70]}")
agg = {}
for w, wi, n, s in res:
    op = s.split()[1] if s.startswith("@") else s.split()[0]
    a = agg.setdefault(op, [0, 0, 0])
    a[0] += w; a[1] += wi; a[2] += n
print("by opcode (wavefronts, ideal, instructions):")
for op, (w, wi, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {op:16s} {w / 1e6:8.2f}M ideal {wi / 1e6:7.2f}M inst {n / 1e6:7.2f}M  per-inst {w / max(n, 1):5.2f}")
