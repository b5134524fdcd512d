#!/bin/bash
# K1 variants (compat / philox / philox frozen / philox at 768 threads), then GPU tests
mkdir -p gpurun_out
for r in 0 1; do timeout 120 ./tools/bin/k1bench 10000000000 5 $r 0; done 2>&1 | tee gpurun_out/k1bench.txt
timeout 120 ./tools/bin/k1bench 10000000000 5 1 1 2>&1 | tee -a gpurun_out/k1bench.txt
timeout 120 ./tools/bin/k1bench_p768 10000000000 5 1 0 2>&1 | tee -a gpurun_out/k1bench.txt
timeout 120 ./tools/bin/k1bench 1000000000 5 1 0 2>&1 | tee -a gpurun_out/k1bench.txt
if [ "${SKIP_TESTS:-0}" = "0" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -15 gpurun_out/pytest_gpu.txt
fi
