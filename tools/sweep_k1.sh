#!/bin/bash
# kernel-1 shapes on C3 / C4 with the current build, plus the u1 build (1-op batches at P = 4)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
for cfg in "C3 128 4 1 768" "C3 64 2 1 768" "C3 128 4 1 704" "C4 128 2 1 768" "C4 64 1 1 768" "C4 128 4 1 384" "C4 128 1 1 768"; do
  set -- $cfg
  cyc=300; [ $1 = C4 ] && cyc=10
  timeout 400 python bench.py --config $1 --lane-tile $2 --cluster $3 --kernel $4 --threads $5 --cycles $cyc --steps 2 --warmup 3 --no-e2e --no-cpu 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$cfg', round(d['ms_per_step']/$cyc*1e3,2), 'us/cycle frac', round(d['roofline']['frac'],3), d['config']['launch'])"
done > $O/sweep_k1.txt 2>&1
export RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_u1.so
for c in C3 C4; do
  cyc=300; [ $c = C4 ] && cyc=10
  timeout 400 python bench.py --config $c --cycles $cyc --steps 2 --warmup 3 --no-e2e --no-cpu 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('u1 $c', round(d['ms_per_step']/$cyc*1e3,2), 'us/cycle frac', round(d['roofline']['frac'],3), d['config']['launch'])"
done >> $O/sweep_k1.txt 2>&1
