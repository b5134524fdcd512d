#!/bin/bash
mkdir -p gpurun_out
for b in k1bench k1bench_p1024; do echo -n "$b: "; timeout 60 ./tools/bin/$b 10000000000 3 1 0 4 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -4 gpurun_out/pytest_gpu.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vsample_kernel --launch-skip 4 -c 1 -o gpurun_out/k1_bench_r01d python bench.py --steps 2 --warmup 3 --no-cpu --no-compat > gpurun_out/ncu_k1b.log 2>&1; tail -1 gpurun_out/ncu_k1b.log
