#!/bin/bash
mkdir -p gpurun_out; OUT=gpurun_out/latc.txt; : > $OUT
for round in 1 2; do for c in ${CS:-8 4 2 1}; do
  echo "== copies<=$c" | tee -a $OUT
  timeout 60 ./tools/bin/latbench_c$c fixed 2>&1 | tee -a $OUT
  timeout 60 ./tools/bin/latbench_c$c graph 2>&1 | tee -a $OUT
  for r in 1 0; do timeout 60 ./tools/bin/latbench_c$c $r 2>&1 | tail -2 | tee -a $OUT; done
done; done
