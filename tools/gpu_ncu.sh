#!/bin/bash
# ncu evidence: one --set full capture of K1 (philox + compat) via k1bench, and
# the launch list of the default bench command (gpu__time_duration per kernel)
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vsample_kernel -c 1 -o gpurun_out/k1_philox_$TAG ./tools/bin/k1bench 1000000000 1 1 0 > gpurun_out/ncu_k1p.log 2>&1; tail -1 gpurun_out/ncu_k1p.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vsample_kernel -c 1 -o gpurun_out/k1_compat_$TAG ./tools/bin/k1bench 1000000000 1 0 0 > gpurun_out/ncu_k1c.log 2>&1; tail -1 gpurun_out/ncu_k1c.log
if [ "${LAUNCHES:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-compat > gpurun_out/ncu_bench.log 2>&1; tail -2 gpurun_out/ncu_bench.log
fi
