#!/bin/bash
# the reference's acceptance criteria c2-c6 on both streams, plus gate pass rates over seed blocks
mkdir -p gpurun_out
( python -m paper_2202_01753_b200.acceptance compat philox; python -m paper_2202_01753_b200.acceptance rates compat philox ) > gpurun_out/acceptance.txt 2>&1
cat gpurun_out/acceptance.txt
timeout 1500 python -m pytest tests/test_gpu_acceptance.py -q -p no:cacheprovider 2>&1 | tail -3
