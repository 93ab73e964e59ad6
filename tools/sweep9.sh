#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
for lib in librtlsim.so librtlsim_t1024.so; do
export RTLSIM_LIB=paper_2601_18140_b200/lib/$lib
for cfg in "C2 32 4 2" "C2 8 1 2" "C2 16 2 2" "C3 128 4 1"; do
  set -- $cfg
  cyc=1000; [ $1 = C3 ] && cyc=100
  timeout 300 python bench.py --config $1 --lane-tile $2 --cluster $3 --kernel $4 --cycles $cyc --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 \
   | python -c "import json,sys; L=sys.stdin.readlines(); 
try:
  d=json.loads(L[-1]); print('$lib $cfg', round(d['ms_per_step']/$cyc*1e3,2), 'us/cycle frac', round(d['roofline']['frac'],3), d['config']['launch'])
except Exception as e: print('$cfg', 'FAILED', L[-3:])"
done; done > $O/sweep9.txt 2>&1
