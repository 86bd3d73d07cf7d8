mkdir -p gpurun_out
export DROTB_NO_GRAPHS=1
for sz in 10000 500; do
timeout 600 ncu --metrics gpu__time_duration.sum,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/iter_ncu_$sz.csv python scripts/probe_iter_ncu.py $sz > /dev/null 2>&1
python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/iter_ncu_$sz.csv")))
h=None
for r in rows:
    if r and r[0]=="ID": h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r))
        print($sz, d["Kernel Name"][:60], d["Metric Name"], d["Metric Value"])
PY
done
