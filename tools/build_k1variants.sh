#!/bin/bash
# Build k1bench variants (tools/bin/k1bench_<name>) from "name:-Dflags" pairs, in parallel.
cd "$(dirname "$0")/.." || exit 1
mkdir -p tools/bin
FLAGS="-std=c++20 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -Xcompiler -ffp-contract=off -Iinclude"
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  nvcc $FLAGS $defs -o tools/bin/k1bench_$name tools/k1bench.cu -Xptxas -v > tools/bin/k1bench_$name.log 2>&1 &
done
wait
for spec in "$@"; do name=${spec%%:*}; echo "$name: $(grep -A1 'vsample_kernel.*F4.*Li8ELNS1_7RngKindE1ELi50' tools/bin/k1bench_$name.log | grep -o 'Used [0-9]* registers.*' | head -1)"; done
