#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_single -s 3 -c 1 -o $O/single_C1 -f \
   python bench.py --config C1 --steps 1 --warmup 3 --cycles 200 --no-cpu --no-e2e > $O/ncu_single_C1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_single -s 3 -c 1 -o $O/single_C5 -f \
   python bench.py --config C5 --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e > $O/ncu_single_C5.log 2>&1
timeout 300 python bench.py --config C1 --cycles 2000 --steps 3 --no-e2e --no-cpu --no-hash > $O/c1_nohash.json 2>/dev/null
