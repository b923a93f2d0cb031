#!/bin/bash
# Round-2 first GPU check: full GPU parity suite, default bench (configs[3]), reference arm.
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv > gpurun_out/nvsmi_r2a.txt 2>&1
nproc >> gpurun_out/nvsmi_r2a.txt
timeout 900 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo "rc=$?" >> gpurun_out/bench_r2a.err
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_r2a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2a.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r2a_ref.json 2> gpurun_out/bench_r2a_ref.err; echo "rc=$?" >> gpurun_out/bench_r2a_ref.err
