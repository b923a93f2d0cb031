#!/bin/bash
# GPU parity tests, then the bench under several environment settings (kernel time only).
# Usage: bash scripts/gpu_env_ab.sh <tag> "ENV=.. ENV=.." "ENV=.." ...
TAG=${1:-envab}; shift
mkdir -p gpurun_out
cd "$(dirname "$0")/.." || exit 1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
: > gpurun_out/envab_$TAG.txt
for cfg in "" "$@"; do
  r=$(env $cfg timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-clocks 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["kernel_ms"],4), round(d["value"]/1e9,3), d["device_vs_e2e_decisions_identical"])')
  echo "[$cfg] $r" >> gpurun_out/envab_$TAG.txt
done
