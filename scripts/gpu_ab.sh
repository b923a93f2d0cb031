#!/bin/bash
# A/B the kernel variants in paper_2004_08177_b200/lib/var/*.so against lib/libgdvfs.so (bench only).
# Usage: bash scripts/gpu_ab.sh <tag> [bench args...]
TAG=${1:-ab}; shift
mkdir -p gpurun_out
cd "$(dirname "$0")/.." || exit 1
echo "base $(timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-clocks "$@" 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(d["kernel_ms"], d["value"])')" > gpurun_out/ab_$TAG.txt
for v in paper_2004_08177_b200/lib/var/*.so; do
  echo "$(basename $v) $(GDVFS_LIB=$PWD/$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-clocks "$@" 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(d["kernel_ms"], d["value"])')" >> gpurun_out/ab_$TAG.txt
done
