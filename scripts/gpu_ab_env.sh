#!/bin/bash
# A/B of walk-geometry knobs on the configs[3] slice: parity subset first, then one bench line per env setting.
TAG=${1:-ab}; APPS=${2:-200000}
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "${PYTEST_K:-deep or fuzz or k2_grid or internal}" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
i=0
for ENVS in "" ${AB_ENVS}; do
  i=$((i+1))
  env $ENVS timeout 600 python bench.py --apps $APPS --no-extras --no-cpu-baseline --no-clocks --steps 2 --warmup 1 --e2e-steps 1 > gpurun_out/ab_${TAG}_$i.json 2> gpurun_out/ab_${TAG}_$i.err
  echo "$i $ENVS" >> gpurun_out/ab_${TAG}_index.txt
done
