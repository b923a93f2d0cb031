#!/bin/bash
# Parity (new kernels + training) then C4-slice / C2 bench lines.
TAG=${1:-r2d}
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_parity.py -m gpu -x -q --timeout 600 -p no:cacheprovider -k "${PYTEST_K:-train or deep or fuzz or k2_grid or internal or edge}" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --apps 200000 --no-extras --no-cpu-baseline --no-clocks --steps 2 --warmup 1 --e2e-steps 1 > gpurun_out/bench_${TAG}_c4s.json 2> gpurun_out/bench_${TAG}_c4s.err
timeout 600 python bench.py --config c2 --no-extras --no-cpu-baseline --no-clocks --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err
