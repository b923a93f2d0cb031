cd $GRAFT_REPO_ROOT
# Usage: bash scripts/c3ab.sh   (configs[2] under several walk-window settings + the default config)
for cfg in "" "GDVFS_WIN_NODES=1024" "GDVFS_WIN_NODES=2048"; do
  r=$(env $cfg timeout 600 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --no-clocks 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["kernel_ms"],2), d["kernels_ms"], d["device_vs_e2e_decisions_identical"])')
  echo "[$cfg] $r" >> gpurun_out/c3ab.txt
done
r=$(timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-clocks 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["kernel_ms"],4), d["kernels_ms"])')
echo "[c2] $r" >> gpurun_out/c3ab.txt
