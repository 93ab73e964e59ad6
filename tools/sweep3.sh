#!/bin/bash
# kernel 1 (tile-interleaved, P = LT/32) launch shapes vs kernel 2; quick parity first.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c2_structure or c3_structure or fuzz or paper or closed or threads" > $O/pytest_k.log 2>&1; echo "rc=$?" >> $O/pytest_k.log
for cfg in "C2 64 8 1" "C2 32 4 1" "C2 64 4 1" "C2 128 8 1" "C2 32 4 2" "C3 128 4 1" "C3 64 2 1" "C3 128 2 1" "C3 64 1 1" "C3 32 1 1" "C3 32 1 2"; do
  set -- $cfg
  cyc=1000; [ $1 = C3 ] && cyc=100
  timeout 300 python bench.py --config $1 --lane-tile $2 --cluster $3 --kernel $4 --cycles $cyc --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$cfg', round(d['ms_per_step']/$cyc*1e3,2), 'us/cycle frac', round(d['roofline']['frac'],3), d['config']['launch'])"
done > $O/sweep3.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/k1_C3 -f \
   python bench.py --config C3 --kernel 1 --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e > $O/ncu_k1_C3.log 2>&1
echo done
