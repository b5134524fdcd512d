#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list, ncu full capture of K1.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -15 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --maxcalls 1000000000 > /dev/null 2> gpurun_out/ncu1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vsample_kernel -s 2 -c 1 -o gpurun_out/prof_k1 python bench.py --steps 1 --warmup 3 --no-cpu --maxcalls 1000000000 > /dev/null 2> gpurun_out/ncu2.err
ls -la gpurun_out
