#!/bin/bash
# Round evidence: bench line, ncu launch list of the bench command, and one
# ncu --set full capture of K1 inside the bench loop (adapted grid: the 5th
# iteration) for each stream: philox r24 (headline), philox exact bins, compat.
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 300 gpurun_out/bench_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary > gpurun_out/ncu_launch_$TAG.log 2>&1; tail -c 200 gpurun_out/ncu_launch_$TAG.log
for spec in "philox --bins r24" "philox --bins exact" "compat"; do
  name=$(echo $spec | tr -d ' -')
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:vsample_kernel --launch-skip 4 -c 1 -o gpurun_out/k1_${name}_$TAG python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary --rng $spec > gpurun_out/ncu_k1_${name}_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k1_${name}_$TAG.log
done
