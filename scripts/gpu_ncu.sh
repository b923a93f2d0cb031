#!/bin/bash
# ncu evidence for the current build: launch list of one bench run + one --set full capture of the walk and accumulate kernels.
TAG=${1:-n}
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-clocks \
    > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grid_(walk|acc)" -s 6 -c 2 \
    -o gpurun_out/prof_grid_$TAG -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-clocks \
    > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full_$TAG.log
