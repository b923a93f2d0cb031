#!/bin/bash
# A/B: bench lines (kernel times) for several (library, env) variants on several configs.
# Usage: VARIANTS="label:ENV=..;ENV=.. label2:GDVFS_LIB=..." CONFIGS="c4s c2 c2t" bash scripts/gpu_abv.sh <tag>
TAG=${1:-abv}
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
out=gpurun_out/abv_$TAG.txt; : > $out
for cfg in ${CONFIGS:-c4s c2 c2t}; do
  for v in base:X=1 ${VARIANTS}; do
    label=${v%%:*}; envs=${v#*:}; envs=${envs//;/ }
    if [ "$cfg" = c4s ]; then args="--apps ${APPS:-200000} --steps 3 --warmup 1"; else args="--config $cfg --steps 5 --warmup 3"; fi
    r=$(env $envs timeout 600 python bench.py $args --no-extras --no-cpu-baseline --no-clocks --e2e-steps 1 2>>gpurun_out/abv_$TAG.err | python scripts/abv_line.py 2>&1)
    echo "$cfg $label: $r" >> $out
  done
done
