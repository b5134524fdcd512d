#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider 2>&1 | tail -5
MCB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --maxcalls 100000000 > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
tail -3 gpurun_out/bench_2rank.err; python -c "import json; d=json.load(open('gpurun_out/bench_2rank.json')); print(d['value'], d['n_gpus'], d.get('time_to_epsrel'))"
python bench.py --impl reference --steps 3 --warmup 3 | cut -c1-600
