#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cli.py -q -p no:cacheprovider 2>&1 | tail -3
timeout 1500 python bench.py --suite gpurun_out/suite.jsonl 2> gpurun_out/suite.err; echo "suite rc=$?"
tail -2 gpurun_out/suite.err
wc -l gpurun_out/suite.jsonl
