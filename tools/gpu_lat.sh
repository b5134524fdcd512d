#!/bin/bash
mkdir -p gpurun_out
python tools/latency.py 2>&1 | tee gpurun_out/latency.txt
if [ "${SKIP_TESTS:-0}" = "0" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -4 gpurun_out/pytest_gpu.txt
fi
