#!/bin/bash
# ncu --set full of one k_lanes* launch: ncu_one.sh NAME bench-args...
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; N=$1; shift
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/$N -f \
   python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e "$@" > $O/ncu_$N.log 2>&1
