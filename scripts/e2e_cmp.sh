#!/bin/bash
# e2e (host buffers) with and without the streamed batch uploads, on a 2M-app configs[3] slice, after a parity subset.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "streamed or internal or c2_full or deep_config" > gpurun_out/pytest_p16.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_p16.log
for e in 1 0; do
  GDVFS_STREAM_INPUTS=$e timeout 900 python bench.py --apps 2000000 --steps 3 --warmup 1 --e2e-steps 3 --no-extras --no-cpu-baseline --no-clocks 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('stream=$e', round(d['ms_per_step'],1), 'e2e', round(d['e2e']['ms_per_step'],1), d['device_vs_e2e_decisions_identical'])" >> gpurun_out/e2ecmp.txt
done
