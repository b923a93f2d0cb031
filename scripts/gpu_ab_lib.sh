#!/bin/bash
# A/B of library builds (GDVFS_LIB) on the configs[3] slice and configs[1]: one bench line each.
TAG=${1:-abl}; shift
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
rm -f gpurun_out/ab_${TAG}_index.txt
i=0
for LIB in default "$@"; do
  for CFG in "--apps 200000" "--config c2"; do
    i=$((i+1))
    if [ "$LIB" = default ]; then E=""; else E="GDVFS_LIB=$LIB"; fi
    env $E timeout 600 python bench.py $CFG --no-extras --no-cpu-baseline --no-clocks --steps 3 --warmup 2 --e2e-steps 1 > gpurun_out/ab_${TAG}_$i.json 2> gpurun_out/ab_${TAG}_$i.err
    echo "$i $LIB $CFG" >> gpurun_out/ab_${TAG}_index.txt
  done
done
