#!/bin/bash
# Parity subset then variant A/B: bash scripts/gpu_iter3.sh TAG  (PYTEST_K, VARIANTS, CONFIGS, APPS from env)
TAG=${1:-it}
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
bash scripts/gpu_abv.sh $TAG
