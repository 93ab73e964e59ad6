#!/bin/bash
# Kernel 7 A/B: record prefetch one op ahead.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
B="python bench.py --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
timeout 600 $B > $O/p_base.json 2>&1
RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_rp.so RTLSIM_AUTOBUILD=0 timeout 600 $B > $O/p_rp.json 2>&1
timeout 600 $B > $O/p_base2.json 2>&1
echo done
