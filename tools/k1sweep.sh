#!/bin/bash
./tools/bin/dexp_check
for r in 1 0; do echo -n "rng $r: "; timeout 60 ./tools/bin/k1bench 10000000000 3 $r 0 4 | tail -1; done
