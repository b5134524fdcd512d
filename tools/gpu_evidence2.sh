#!/bin/bash
# ncu captures summarised ON the box (the .ncu-rep files are too large to
# bring back): launch list + one --set full capture of K1 per stream.
mkdir -p gpurun_out/ncu
TAG=${TAG:-r02}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary > gpurun_out/ncu_launch_$TAG.log 2>&1; tail -c 200 gpurun_out/ncu_launch_$TAG.log
EVALS=859963392
for spec in "philox --bins r24" "philox --bins exact" "compat"; do
  name=$(echo $spec | tr -d ' -')
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:vsample_kernel --launch-skip 4 -c 1 -o /tmp/k1_${name}_$TAG python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary --rng $spec > gpurun_out/ncu_k1_${name}_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k1_${name}_$TAG.log
  python tools/summarize_ncu.py /tmp/k1_${name}_$TAG.ncu-rep gpurun_out/launches_$TAG.csv ${TAG}_${name} $EVALS > gpurun_out/sum_${name}.txt 2>&1
  ncu -i /tmp/k1_${name}_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu/src_${name}.csv 2>/dev/null
  ncu -i /tmp/k1_${name}_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu/raw_${name}.csv 2>/dev/null
  gzip -f gpurun_out/ncu/src_${name}.csv
done
cp profiles/ncu_k1_${TAG}_* profiles/launches_${TAG}_* profiles/k1_traffic.json gpurun_out/ncu/ 2>/dev/null
ls -la gpurun_out/ncu
