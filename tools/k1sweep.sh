#!/bin/bash
./tools/bin/latbench 1 1000000 5
