#!/bin/bash
# Launch-shape sweep with the 640-thread build: "config lane_tile cluster kernel threads"
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
for cfg in "C2 32 8 2 320" "C2 32 8 2 288" "C2 32 8 2 256" "C2 16 8 2 320" "C2 32 4 2 320" "C2 32 4 2 640"; do
  set -- $cfg
  cyc=1000; [ $1 = C3 ] && cyc=300
  timeout 300 python bench.py --config $1 --lane-tile $2 --cluster $3 --kernel $4 --threads $5 --cycles $cyc --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$cfg', round(d['ms_per_step']/$cyc*1e3,2), 'us/cycle frac', round(d['roofline']['frac'],3), d['config']['launch'])"
done > $O/sweep640.txt 2>&1
