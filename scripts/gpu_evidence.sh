#!/bin/bash
# Round evidence: GPU suite + smoke, the default bench line (configs[3], 10M apps), its ncu launch list and one
# `ncu --set full` capture of the walk + accumulate kernels of the same command.
TAG=${1:-ev}
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline --no-clocks --e2e-steps 1 \
    > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/ncu_launch_$TAG.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"grid_(walk|acc)" -s 600 -c 2 \
    -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-clocks --e2e-steps 1 \
    > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/ncu_full_$TAG.log
