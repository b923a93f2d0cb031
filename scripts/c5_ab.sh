#!/bin/bash
# configs[4] latency probe for the library variants in paper_2004_08177_b200/lib/var/*.so (and the default build).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
{ echo "base: $(python scripts/c5_probe.py 2>&1 | grep 'B=64: wall')"
  for v in paper_2004_08177_b200/lib/var/*.so; do
    echo "$(basename $v): $(GDVFS_LIB=$PWD/$v python scripts/c5_probe.py 2>&1 | grep 'B=64: wall')"
  done; } > gpurun_out/c5_ab.txt 2>&1
