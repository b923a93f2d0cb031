#!/bin/bash
# configs[0] C++ drop-in (facade_test --bench) under several GDVFS_* settings: bash scripts/c1bisect.sh [reps] [jobs]
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
for e in "X=1" "GDVFS_WIDE=0" "X=2" "GDVFS_BATCH_BYTES=2147483648" "GDVFS_WALK_SPLIT_MAJOR=0"; do
  echo "== $e: $(env $e integration/_build/facade_test --bench ${1:-9} 100 10 ${2:-1000} 2>&1 | tail -1 | cut -c1-300)"
done > gpurun_out/c1bisect.txt 2>&1
