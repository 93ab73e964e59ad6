#!/bin/bash
# Kernel 6 occupancy experiment: P = 2 (64-lane tiles) at 768 vs 1024 threads, P = 4 at 768.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
B="timeout 600 python bench.py --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
N="RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_nopf.so RTLSIM_AUTOBUILD=0"
T="RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_t1024.so RTLSIM_AUTOBUILD=0"
env $N $B --kernel 6 --lane-tile 64 --threads 768 > $O/occ_p2_t768.json 2>&1
env $T $B --kernel 6 --lane-tile 64 --threads 1024 > $O/occ_p2_t1024.json 2>&1
env $N $B --kernel 6 --lane-tile 64 --threads 512 > $O/occ_p2_t512.json 2>&1
env $N $B --kernel 6 --lane-tile 128 --threads 512 > $O/occ_p4_t512.json 2>&1
env $N $B --kernel 6 --lane-tile 128 --threads 768 --cluster 8 > $O/occ_p4_t768_c8.json 2>&1
env $N $B --kernel 1 --lane-tile 64 --threads 768 > $O/occ_k1_p2_t768.json 2>&1
echo done
