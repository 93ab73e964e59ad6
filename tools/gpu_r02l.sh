#!/bin/bash
# Kernel 7 (record-based lane kernel) bring-up: parity on the lane tests, C3 bench vs kernel 1, ncu capture.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_passes.py -m gpu -q -x -p no:cacheprovider \
  -k "kernel7 or kernel-7 or 7 or c3_structure or fuzz_corpus" > $O/pytest_l.log 2>&1; echo "pytest rc=$?" >> $O/pytest_l.log
B="python bench.py --config C3 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 600 $B --kernel 7 > $O/k7_C3.json 2>&1
timeout 600 $B --kernel 1 > $O/k1_C3.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C3_k7 -f \
   python bench.py --kernel 7 --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e --no-hash-off-pass > $O/ncu_full_C3_k7.log 2>&1
echo done
