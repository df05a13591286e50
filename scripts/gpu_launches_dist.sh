# ncu launch list (device time per kernel) of one 200M sort of $DIST (second call).
make -j8 > gpurun_out/make.log 2>&1 || exit 1
P="python scripts/prof_sort.py --dist ${DIST:-telemetry} --n 200000000 --reps 2"
LS_GRAPH=0 $P > gpurun_out/prof_plain.log 2>&1 && \
LS_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${DIST:-telemetry}.csv $P > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?"
python - <<'PY'
import csv, os
d=os.environ.get("DIST","telemetry")
rows=list(csv.reader(open(f"gpurun_out/launches_{d}.csv")))
hdr=next(r for r in rows if r and r[0]=="ID")
out=[]
for r in rows:
    if len(r)==len(hdr) and r[0]!="ID":
        x=dict(zip(hdr,r))
        if x["Metric Name"]=="gpu__time_duration.sum":
            out.append((x["Kernel Name"].split("(")[0][:50], float(x["Metric Value"].replace(",",""))))
half=len(out)//2
for n,v in out[half:]: print(f"{n:50s} {v}")
PY
