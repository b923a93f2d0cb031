#!/bin/bash
# Cost split experiment: kernel time vs the fraction of clock splits in the trees.
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
for w in 0.0 0.01 0.04 0.1; do
  echo "w_clk=$w $(timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-clocks --w-clk $w 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(d["kernel_ms"], d["value"])')" >> gpurun_out/wclk_$1.txt
done
