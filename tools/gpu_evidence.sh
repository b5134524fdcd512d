#!/bin/bash
# Round evidence: bench line, ncu launch list of the bench command, one ncu
# --set full capture of K1 inside the bench loop (adapted grid), and the same
# for the compat stream.
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 400 gpurun_out/bench_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-compat > gpurun_out/ncu_launch_$TAG.log 2>&1; tail -c 200 gpurun_out/ncu_launch_$TAG.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vsample_kernel --launch-skip 4 -c 1 -o gpurun_out/k1_philox_$TAG python bench.py --steps 2 --warmup 3 --no-cpu --no-compat > gpurun_out/ncu_k1p_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k1p_$TAG.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vsample_kernel --launch-skip 4 -c 1 -o gpurun_out/k1_compat_$TAG python bench.py --steps 2 --warmup 3 --no-cpu --no-compat --rng compat > gpurun_out/ncu_k1c_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k1c_$TAG.log
