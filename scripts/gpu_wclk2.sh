#!/bin/bash
# Kernel split vs the clock-split rate of the synthetic trees (configs[1] shape).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
: > gpurun_out/wclk2.txt
for w in 0 0.02 0.04 0.08; do
  r=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-clocks --w-clk $w 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["kernel_ms"],4), {k: round(v,4) for k,v in d["kernels_ms"].items()}, round(d["binding_roofline"]["frac"],3))')
  echo "w_clk=$w $r" >> gpurun_out/wclk2.txt
done
