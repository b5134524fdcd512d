#!/bin/bash
# Round-2 evidence after a K1 change: latency, GPU tests, bench line, ncu (launch list + K1 per stream).
mkdir -p gpurun_out
python tools/latency.py > gpurun_out/latency.txt 2>&1; cat gpurun_out/latency.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -3 gpurun_out/pytest_gpu.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
TAG=${TAG:-r02e} bash tools/gpu_evidence2.sh > gpurun_out/evidence.log 2>&1; tail -5 gpurun_out/evidence.log
