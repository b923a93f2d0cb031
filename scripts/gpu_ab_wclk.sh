#!/bin/bash
# A/B the library variants in lib/var/*.so at several clock-split rates.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out; : > gpurun_out/ab_wclk.txt
for w in 0.04 0.08; do
  for v in base paper_2004_08177_b200/lib/var/*.so; do
    if [ "$v" = base ]; then envv=""; else envv="GDVFS_LIB=$PWD/$v"; fi
    r=$(env $envv timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-clocks --w-clk $w 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["kernel_ms"],4), {k: round(v,4) for k,v in d["kernels_ms"].items()})')
    echo "w=$w $(basename $v) $r" >> gpurun_out/ab_wclk.txt
  done
done
