#!/bin/bash
# K1 philox threads sweep (k1bench_p<threads> built with -DMCB_SAMPLE_THREADS_PHILOX)
for b in k1bench_p768 k1bench_p896 k1bench_p1024; do
  for mc in 10000000000 1000000000; do timeout 120 ./tools/bin/$b $mc 5 1 0; done
done
timeout 120 ./tools/bin/k1bench_p768 10000000000 5 0 0
