#!/bin/bash
# Parity suite + C4-slice and C2 bench lines for the current build.
TAG=${1:-r2c}
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --apps 200000 --no-extras --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/bench_${TAG}_c4s.json 2> gpurun_out/bench_${TAG}_c4s.err
timeout 600 python bench.py --config c2 --no-extras --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err
