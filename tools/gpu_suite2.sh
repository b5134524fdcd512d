#!/bin/bash
# BASELINE configs 1-5 beside the reference CPU library, and the C5 scale sweep with CPU columns.
mkdir -p gpurun_out
timeout 2400 python bench.py --suite gpurun_out/suite_${TAG:-r02}.jsonl > gpurun_out/suite.log 2>&1; echo "suite rc=$?"
timeout 1200 python bench.py --scale gpurun_out/scale_${TAG:-r02}.csv > gpurun_out/scale.log 2>&1; echo "scale rc=$?"
tail -3 gpurun_out/scale.log
