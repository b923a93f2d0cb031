#!/bin/bash
# Full GPU parity suite + the C1 production-path bench line.
TAG=${1:-full}
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 900 python bench.py --config c1 --steps 5 > gpurun_out/bench_${TAG}_c1.json 2> gpurun_out/bench_${TAG}_c1.err
timeout 900 python bench.py --config c1 --apps 1000 --steps 3 > gpurun_out/bench_${TAG}_c1k.json 2>> gpurun_out/bench_${TAG}_c1.err
