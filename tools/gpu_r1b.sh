#!/bin/bash
# round-1 session B: philox fast path first measurement
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for r in 0 1; do timeout 120 ./tools/bin/k1bench 10000000000 5 $r 0; done 2>&1 | tee gpurun_out/k1bench.txt
timeout 120 ./tools/bin/k1bench 10000000000 5 1 1 2>&1 | tee -a gpurun_out/k1bench.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -15 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vsample_kernel -c 1 -o gpurun_out/k1_philox ./tools/bin/k1bench 1000000000 1 1 0 > gpurun_out/ncu_k1.log 2>&1
tail -2 gpurun_out/ncu_k1.log
