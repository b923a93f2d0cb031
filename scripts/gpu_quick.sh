#!/bin/bash
# Fast iteration loop on the GPU box: GPU parity tests, kernel bench, one ncu --set full capture.
# Usage: bash scripts/gpu_quick.sh <tag> [bench args...]
TAG=${1:-q}
shift
mkdir -p gpurun_out
cd "$(dirname "$0")/.." || exit 1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grid_(walk|acc)" -s 6 -c 2 \
    -o gpurun_out/prof_grid_$TAG -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-clocks "$@" \
    > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full_$TAG.log
