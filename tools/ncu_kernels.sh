#!/bin/bash
# per-kernel durations of one command (measurement tool): bash tools/ncu_kernels.sh CMD...
ncu --metrics gpu__time_duration.sum --clock-control none --csv "$@" 2>/dev/null > gpurun_out/_k.csv
python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/_k.csv")))
h=[r for r in rows if "Kernel Name" in r][0]
for r in rows:
    if len(r)==len(h) and r!=h:
        d=dict(zip(h,r)); print(d["Kernel Name"][:48], d["Grid Size"], d["Metric Value"], d["Metric Unit"])
PY
