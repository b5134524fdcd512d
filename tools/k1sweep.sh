#!/bin/bash
for b in k1bench k1bench_p1024; do echo -n "$b: "; ./tools/bin/$b 10000000000 3 1 0 4 | tail -1; done
echo -n "frozen adapted: "; ./tools/bin/k1bench 10000000000 3 1 1 4 | tail -1
