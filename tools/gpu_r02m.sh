#!/bin/bash
# Kernel 7 with op pairs (default build) vs without; parity subset; C3 at 4096 / 2048 lanes, C4.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_passes.py -m gpu -q -x -p no:cacheprovider \
  -k "kernel7 or kernel-7 or 7 or c3_structure or fuzz_corpus" > $O/pytest_m.log 2>&1; echo "pytest rc=$?" >> $O/pytest_m.log
B="python bench.py --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
N="RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_nopairs.so RTLSIM_AUTOBUILD=0"
timeout 600 $B --kernel 7 > $O/m_k7_pairs.json 2>&1
env $N timeout 600 $B --kernel 7 > $O/m_k7_nopairs.json 2>&1
timeout 600 $B --kernel 7 --lanes 2048 > $O/m_k7_2048.json 2>&1
timeout 600 $B --kernel 1 --lanes 2048 > $O/m_k1_2048.json 2>&1
timeout 900 python bench.py --config C4 --cycles 20 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 7 > $O/m_k7_C4.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C3_k7 -f \
   python bench.py --kernel 7 --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e --no-hash-off-pass > $O/ncu_full_C3_k7.log 2>&1
echo done
