#!/bin/bash
# ncu --set full of the K1 launch inside the bench loop (adapted grid, iteration 5)
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vsample_kernel --launch-skip 4 -c 1 -o gpurun_out/k1_bench_$TAG python bench.py --steps 2 --warmup 3 --no-cpu --no-compat > gpurun_out/ncu_k1b.log 2>&1; tail -2 gpurun_out/ncu_k1b.log
