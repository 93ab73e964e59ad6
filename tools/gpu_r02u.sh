#!/bin/bash
# Kernel 7 CTA size A/B: 768 threads (80 registers), 896 (72), 1,024 (64, small spills); C3 and C4.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
B3="python bench.py --config C3 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 7"
B4="python bench.py --config C4 --cycles 20 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 7"
timeout 300 $B3 > $O/u_C3_768.json 2>&1
RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_r896.so RTLSIM_AUTOBUILD=0 timeout 300 $B3 --threads 896 > $O/u_C3_896.json 2>&1
RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_r1024.so RTLSIM_AUTOBUILD=0 timeout 300 $B3 --threads 1024 > $O/u_C3_1024.json 2>&1
timeout 300 $B4 > $O/u_C4_768.json 2>&1
RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_r896.so RTLSIM_AUTOBUILD=0 timeout 300 $B4 --threads 896 > $O/u_C4_896.json 2>&1
RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_r1024.so RTLSIM_AUTOBUILD=0 timeout 300 $B4 --threads 1024 > $O/u_C4_1024.json 2>&1
echo done
