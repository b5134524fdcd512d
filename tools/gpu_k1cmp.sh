#!/bin/bash
# A/B of k1bench builds (tools/bin/k1bench_<name>) interleaved; RNGS: 0 compat, 1 philox, 2 philox exact bins.
mkdir -p gpurun_out; OUT=gpurun_out/k1cmp.txt; : > $OUT
for round in 1 2; do for rng in ${RNGS:-1 0}; do for v in ${VARS:-head tab}; do for mc in ${MCS:-1000000000 10000000000}; do
  line=$(timeout 120 ./tools/bin/k1bench_$v $mc 4 $rng 0 2>&1 | tail -1)
  echo "var=$v $line" | awk '{print $1, $2, $6, $(NF-1), $NF}' | tee -a $OUT
done; done; done; done
