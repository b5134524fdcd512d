#!/bin/bash
# Compare k1bench variants (tools/build_k1variants.sh) on the box: interleaved
# rounds so clock drift hits every variant alike; the estimate bits must agree.
mkdir -p gpurun_out
OUT=gpurun_out/k1var.txt; : > $OUT
VARS=${VARS:-$(ls tools/bin/k1bench_* | grep -v '\.log$' | xargs -n1 basename | sed 's/k1bench_//')}
for round in 1 2 3; do
  for v in $VARS; do
    for mc in 1000000000 10000000000; do
      line=$(timeout 120 ./tools/bin/k1bench_$v $mc 4 ${RNG:-1} 0 2>&1 | tail -1)
      echo "round=$round var=$v maxcalls=$mc $line" | tee -a $OUT
    done
  done
done
