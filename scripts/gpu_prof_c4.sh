#!/bin/bash
# ncu evidence at the configs[3] shape (2000-tree depth-12 E+T, 267 clocks) on a 200k-app slice:
# launch list + one --set full capture of the walk and accumulate kernels.
TAG=${1:-c4}; APPS=${2:-200000}
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --apps $APPS --steps 2 --warmup 1 --no-cpu-baseline --no-clocks --no-extras --e2e-steps 1 \
    > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch_$TAG.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"grid_(walk|acc)" -s 2 -c 2 \
    -o gpurun_out/prof_$TAG -f python bench.py --apps $APPS --steps 1 --warmup 1 --no-cpu-baseline --no-clocks --no-extras --e2e-steps 1 \
    > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full_$TAG.log
