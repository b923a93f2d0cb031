#!/bin/bash
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
for c in 100 80 60 40 20; do
  for w in 0.0 0.04; do
  echo "carve=$c w=$w $(GDVFS_CARVEOUT=$c timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-clocks --w-clk $w 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(d["kernel_ms"], d["value"])')" >> gpurun_out/carve_$1.txt
  done
done
