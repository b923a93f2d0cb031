#!/bin/bash
# GPU parity suite (incl. the multi-device ABI and drop-in variants).
mkdir -p gpurun_out; cd "$(dirname "$0")/.." || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider -k "${1:-}" > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2b.log
for a in "100 10 1000" "100 10 1000 25"; do ./integration/_build/facade_test $a >> gpurun_out/facade_r2b.txt 2>&1; done
