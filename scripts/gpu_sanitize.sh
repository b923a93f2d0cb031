#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_small.py.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_small.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.txt
done
