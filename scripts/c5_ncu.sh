#!/bin/bash
# ncu --set full of the configs[4] walk kernel: this build and the round-1 worktree (_r1/, if present).
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grid_walk -s 40 -c 1 -o gpurun_out/prof_c5now -f python scripts/c5_probe.py > gpurun_out/ncu_c5now.log 2>&1
cd _r1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:grid_walk -s 40 -c 1 -o ../gpurun_out/prof_c5r1 -f python scripts/c5_probe.py > ../gpurun_out/ncu_c5r1.log 2>&1
