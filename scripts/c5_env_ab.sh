#!/bin/bash
# configs[4] latency probe under several environment settings.
# Usage: bash scripts/c5_env_ab.sh <tag> "ENV=.. ENV=.." ...
TAG=${1:-c5ab}; shift
mkdir -p gpurun_out
cd "$(dirname "$0")/.." || exit 1
: > gpurun_out/c5ab_$TAG.txt
for cfg in "" "$@"; do
  echo "[$cfg] $(env $cfg timeout 300 python scripts/c5_probe.py 64 2>&1 | head -1)" >> gpurun_out/c5ab_$TAG.txt
done
