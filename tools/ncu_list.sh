#!/bin/bash
# usage: tools/ncu_list.sh <python args...>  -- per-launch durations (ncu, cold-cache) of our kernels
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l.csv python "$@" > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/l.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:]:
    if "bcg::" in r[ki] and "probe" not in r[ki]: print(r[ki].split("(")[0][:50], float(r[vi].replace(",",""))/1e6)
PY
