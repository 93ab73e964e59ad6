#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_single2 -s 3 -c 1 -o $O/prof_single_C5 -f \
   python bench.py --config C5 --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e > $O/ncu_single_C5.log 2>&1
