#!/bin/bash
mkdir -p gpurun_out
./tools/bin/k1_768 1000000000 5
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -3 gpurun_out/pytest_gpu.txt
python tools/c1_timing.py 2>&1 | tee gpurun_out/c1_timing.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches.csv python tools/c1_only.py > /dev/null 2>&1; python - <<PY
import csv
from collections import defaultdict
rows=list(csv.reader(open("gpurun_out/c1_launches.csv")))
s=next(i for i,r in enumerate(rows) if r and r[0]=="ID")
h=rows[s]; ik=h.index("Kernel Name"); iv=h.index("Metric Value")
d=defaultdict(list)
for r in rows[s+1:]: d[r[ik].split("(")[0][-40:]].append(float(r[iv]))
for k,v in d.items(): print(k, len(v), sum(v)/len(v))
PY
