#!/bin/bash
for b in k1bench; do echo -n "$b: "; timeout 60 ./tools/bin/$b 10000000000 3 1 0 4 | tail -1; done
