#!/bin/bash
# configs[3] evidence: headline bench line at full size + launch list + one ncu --set full of walk / acc at the C4 shape.
# Usage (through gpurun): bash scripts/gpu_c4.sh <tag> [bench args...]
TAG=${1:-c4}; shift
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv > gpurun_out/nvsmi_$TAG.txt 2>&1
nproc >> gpurun_out/nvsmi_$TAG.txt; free -g >> gpurun_out/nvsmi_$TAG.txt
timeout 900 python bench.py "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"grid_(walk|acc)" -s 4 -c 2 \
    -o gpurun_out/prof_c4_$TAG -f python bench.py --apps 20000 --steps 1 --warmup 0 --no-cpu-baseline --no-clocks --no-extras --e2e-steps 1 \
    > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full_$TAG.log
fi
