#!/bin/bash
# Diagnostic: kernel 1 with every operand gather hitting row 0 (L1-resident; wrong results) vs the real build:
# how much of a C3 cycle is exposed gather latency.  Plus the new auto shapes at 2048 / 512 lanes.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
B="python bench.py --config C3 --cycles 500 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 1"
timeout 300 $B > $O/fake_real.json 2>&1
RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_fake.so RTLSIM_AUTOBUILD=0 timeout 300 $B > $O/fake_fake.json 2>&1
RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_fake.so RTLSIM_AUTOBUILD=0 timeout 300 $B --no-hash > $O/fake_fake_nohash.json 2>&1
timeout 300 $B --no-hash > $O/fake_real_nohash.json 2>&1
for l in 2048 512; do timeout 300 python bench.py --config C3 --cycles 500 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --lanes $l > $O/auto_$l.json 2>&1; done
echo done
