#!/bin/bash
# quick GPU check: K1 microbench (compat/philox/philox frozen), GPU tests, bench line
mkdir -p gpurun_out
for r in 0 1; do timeout 120 ./tools/bin/k1bench 10000000000 5 $r 0; done 2>&1 | tee gpurun_out/k1bench.txt
timeout 120 ./tools/bin/k1bench 10000000000 5 1 1 2>&1 | tee -a gpurun_out/k1bench.txt
if [ "${SKIP_TESTS:-0}" = "0" ]; then
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -15 gpurun_out/pytest_gpu.txt
fi
if [ "${SKIP_BENCH:-0}" = "0" ]; then
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
fi
