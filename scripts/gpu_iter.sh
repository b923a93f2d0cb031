#!/bin/bash
# Iteration loop: GPU parity tests (subset or all), then bench lines.
# Usage: bash scripts/gpu_iter.sh <tag> "<pytest -k expr or ALL or NONE>" "<bench args c4>" ["<bench args 2>"]
TAG=${1:-it}; KEXPR=${2:-ALL}; B1=${3:-}; B2=${4:-}
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
if [ "$KEXPR" = "ALL" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
elif [ "$KEXPR" != "NONE" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "$KEXPR" > gpurun_out/pytest_$TAG.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
if [ -n "$B1" ]; then timeout 900 python bench.py $B1 > gpurun_out/bench_${TAG}_1.json 2> gpurun_out/bench_${TAG}_1.err; echo "rc=$?" >> gpurun_out/bench_${TAG}_1.err; fi
if [ -n "$B2" ]; then timeout 900 python bench.py $B2 > gpurun_out/bench_${TAG}_2.json 2> gpurun_out/bench_${TAG}_2.err; echo "rc=$?" >> gpurun_out/bench_${TAG}_2.err; fi
