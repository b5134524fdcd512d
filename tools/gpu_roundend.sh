#!/bin/bash
# What the driver runs at round end: GPU tests, smoke, the reference arm, the bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -3 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --impl reference --steps 10 --warmup 3 2>/dev/null | cut -c1-200
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; python -c "import json; d=json.load(open('gpurun_out/bench_final.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['gpu_launches'], d['clocks'])"
