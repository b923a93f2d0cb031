#!/bin/bash
# One GPU round trip: tests, smoke, bench (both arms), launch list, one ncu --set full capture.
# Usage (from the repo root, through gpurun): bash scripts/gpu_bench.sh [tag]
TAG=${1:-r1}
mkdir -p gpurun_out
cd "$(dirname "$0")/.." || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 ./integration/_build/facade_test > gpurun_out/facade_$TAG.log 2>&1
echo "facade rc=$?" >> gpurun_out/facade_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
echo "ref rc=$?" >> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-clocks > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grid_(walk|acc)" -s 6 -c 2 \
    -o gpurun_out/prof_grid_$TAG -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-clocks \
    > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full_$TAG.log
