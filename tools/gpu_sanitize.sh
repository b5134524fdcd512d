#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small shapes
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.txt
done
