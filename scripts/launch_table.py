"""Per-kernel time of the last sort in an ncu launch-list CSV (prof_sort, reps 2)."""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))]
rows = [r for r in rows if r["Metric Name"] == "gpu__time_duration.sum"]
ks = [(r["Kernel Name"].split("(")[0].replace("void ", "").replace("ls::", "").replace("(int)", ""),
       float(r["Metric Value"]), r["Metric Unit"]) for r in rows]
# keep the second half (the measured rep)
i0 = max(i for i, k in enumerate(ks) if k[0].startswith("k_init"))
agg = OrderedDict()
for name, v, u in ks[i0:]:
    v = v / 1e3 if u in ("ns", "nsecond") else v if u in ("us", "usecond") else v * 1e3
    agg[name] = agg.get(name, 0) + v
tot = sum(agg.values())
for k, v in agg.items():
    print(f"{k:28s} {v:9.1f} us  {100 * v / tot:5.1f}%")
print(f"{'total':28s} {tot:9.1f} us")
