#!/bin/bash
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:finish_kernel --launch-skip 5 -c 1 -o gpurun_out/finish_c1 python tools/c1_only.py philox > gpurun_out/finish_ncu.log 2>&1; tail -1 gpurun_out/finish_ncu.log
ncu --set full --import-source on --clock-control none -k regex:vsample_kernel --launch-skip 5 -c 1 -o gpurun_out/k1_c1 python tools/c1_only.py philox > gpurun_out/k1c1_ncu.log 2>&1; tail -1 gpurun_out/k1c1_ncu.log
