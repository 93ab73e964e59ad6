#!/bin/bash
# Launch-shape sweep for the lane kernel (C2, C3 short runs): ms per cycle.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
for cfg in "C2 8 1" "C2 8 2" "C2 16 1" "C2 16 2" "C2 16 4" "C2 32 2" "C2 32 4" "C2 32 8" "C3 32 1" "C3 16 1" "C3 8 1"; do
  set -- $cfg
  cyc=1000; [ $1 = C3 ] && cyc=100
  timeout 300 python bench.py --config $1 --lane-tile $2 --cluster $3 --cycles $cyc --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$cfg', round(d['ms_per_step']/$cyc*1e3,2), 'us/cycle frac', round(d['roofline']['frac'],3), d['config']['launch'])"
done > $O/sweep.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/k_lanes_C3 -f \
   python bench.py --config C3 --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e > $O/ncu_full_C3.log 2>&1
echo done
