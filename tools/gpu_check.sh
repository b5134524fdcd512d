#!/bin/bash
# GPU tests, latency and the bench line (no ncu): the round's regular check.
mkdir -p gpurun_out
python tools/latency.py > gpurun_out/latency.txt 2>&1; cat gpurun_out/latency.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -3 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['philox_exact_bins']['value'], d['compat']['value'], d['clocks'])"
