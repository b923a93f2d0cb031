#!/bin/bash
# One `ncu --set full` capture of the walk + accumulate kernels (second batch) on a configs[3] slice.
TAG=${1:-p}; APPS=${2:-40000}; CFG=${3:-c4}
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"grid_(walk|acc)" -s 2 -c 2 \
    -o gpurun_out/prof_$TAG -f python bench.py --config $CFG --apps $APPS --steps 1 --warmup 1 --no-cpu-baseline --no-clocks --no-extras --e2e-steps 1 \
    > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full_$TAG.log
