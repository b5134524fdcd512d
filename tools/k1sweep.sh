#!/bin/bash
for b in k1_640 k1_768 k1_1024; do ./tools/bin/$b 1000000000 5; done
