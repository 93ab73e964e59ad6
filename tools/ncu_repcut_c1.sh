#!/bin/bash
# ncu --set full of k_repcut_smem on C1 (auto single-lane choice: one partition)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_repcut_smem -s 3 -c 1 -o $O/prof_repcut_C1 -f \
   python bench.py --config C1 --steps 1 --warmup 3 --cycles 2000 --no-cpu --no-e2e > $O/ncu_repcut_C1.log 2>&1
