#!/bin/bash
# Round-2 GPU check: all GPU tests (incl. row-mode parity, bench N>1), then the bench line.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -32 gpurun_out/pytest_gpu.txt
if [ "${SKIP_BENCH:-0}" = "0" ]; then
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err; head -c 3000 gpurun_out/bench.json
fi
