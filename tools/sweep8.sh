#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c2_structure or c3_structure or fuzz or paper or closed or threads or chunking" > $O/pytest_k.log 2>&1; echo "rc=$?" >> $O/pytest_k.log
for cfg in "C2 32 4 2" "C2 16 2 2" "C2 8 1 2" "C3 128 4 1" "C4 128 2 1"; do
  set -- $cfg
  cyc=1000; [ $1 = C3 ] && cyc=100; [ $1 = C4 ] && cyc=10
  timeout 300 python bench.py --config $1 --lane-tile $2 --cluster $3 --kernel $4 --cycles $cyc --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 \
   | python -c "import json,sys; L=sys.stdin.readlines(); 
try:
  d=json.loads(L[-1]); print('$cfg', round(d['ms_per_step']/$cyc*1e3,2), 'us/cycle frac', round(d['roofline']['frac'],3), d['config']['launch'])
except Exception as e: print('$cfg', 'FAILED', L[-3:])"
done > $O/sweep8.txt 2>&1
bash tools/trace_run.sh
