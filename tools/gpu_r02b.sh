#!/bin/bash
# Kernel 6 (bit-sliced lane kernel) bring-up: its parity tests, then C3 with kernels 1 and 6.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x -k "kernel6 or kernel-6 or edges or c3_structure or ragged or fuzz or chunking or wide_work or staged or checkpoint or sharding or waveform_changes or threads_variants" \
  --deselect tests/test_gpu_full_scope.py -p no:cacheprovider > $O/pytest_k6.log 2>&1; echo "pytest rc=$?" >> $O/pytest_k6.log
timeout 600 python bench.py --kernel 6 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_k6.json 2> $O/bench_C3_k6.err
timeout 600 python bench.py --kernel 1 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_k1.json 2> $O/bench_C3_k1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C3_k6 -f \
   python bench.py --kernel 6 --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e --no-hash-off-pass > $O/ncu_full_C3_k6.log 2>&1
echo done
