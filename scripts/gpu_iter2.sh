#!/bin/bash
# One iteration: full GPU parity suite, then the configs[3] slice, configs[1] and trained configs[1] lines.
TAG=${1:-it}; APPS=${2:-200000}
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --apps $APPS --no-extras --no-cpu-baseline --no-clocks --steps 3 --warmup 1 --e2e-steps 1 > gpurun_out/bench_${TAG}_c4s.json 2> gpurun_out/bench_${TAG}_c4s.err
for c in c2 c2t c3; do
  timeout 600 python bench.py --config $c --no-extras --no-cpu-baseline --no-clocks --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
python scripts/show_bench.py gpurun_out/bench_${TAG}_*.json > gpurun_out/summary_$TAG.txt 2>&1
