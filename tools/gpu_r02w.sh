#!/bin/bash
# Kernel 7: 3-operand ops in two half passes (RS_K7_SPLIT3) at 896 / 1,024 threads vs the default.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
B3="python bench.py --config C3 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
timeout 300 $B3 > $O/w_base.json 2>&1
RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_s896.so RTLSIM_AUTOBUILD=0 timeout 300 $B3 > $O/w_s896.json 2>&1
RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_s1024.so RTLSIM_AUTOBUILD=0 timeout 300 $B3 --threads 1024 > $O/w_s1024.json 2>&1
timeout 300 $B3 > $O/w_base2.json 2>&1
echo done
