#!/bin/bash
mkdir -p gpurun_out
for rng in philox compat; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches_$rng.csv python tools/c1_only.py $rng > /dev/null 2>&1
python - <<PY
import csv
from collections import defaultdict
rows=list(csv.reader(open("gpurun_out/c1_launches_$rng.csv")))
s=next(i for i,r in enumerate(rows) if r and r[0]=="ID")
h=rows[s]; ik=h.index("Kernel Name"); iv=h.index("Metric Value")
d=defaultdict(list)
for r in rows[s+1:]: d[r[ik].split("(")[0][-50:]].append(float(r[iv].replace(",","")))
for k,v in d.items(): print("$rng", k, len(v), "avg ns", sum(v)/len(v))
PY
done
