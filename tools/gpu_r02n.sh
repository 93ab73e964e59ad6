#!/bin/bash
# Kernel 7 A/B: records dealt in blocks of 1 / 2 / 4 / 8 per warp; CTA sizes.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
B="python bench.py --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 7"
timeout 600 $B > $O/n_b1.json 2>&1
for b in 2 4 8; do RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_b$b.so RTLSIM_AUTOBUILD=0 timeout 600 $B > $O/n_b$b.json 2>&1; done
timeout 600 $B --threads 640 > $O/n_t640.json 2>&1
timeout 600 $B --threads 512 > $O/n_t512.json 2>&1
timeout 600 python bench.py --config C4 --cycles 20 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 7 > $O/n_C4_b1.json 2>&1
RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_b4.so RTLSIM_AUTOBUILD=0 timeout 600 python bench.py --config C4 --cycles 20 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 7 > $O/n_C4_b4.json 2>&1
echo done
