#!/bin/bash
# Kernel 7 at 896 threads (single ops) / 768 (pairs): lane parity subset + C3 / C4 / 2,048-lane benches.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_passes.py tests/test_gpu_full_scope.py -m gpu -q -x -p no:cacheprovider \
  -k "kernel7 or kernel-7 or 7 or c3_structure or fuzz_corpus or wide_work or auto_kernel or threads_variants or c3_full" > $O/pytest_v.log 2>&1; echo "pytest rc=$?" >> $O/pytest_v.log
run() { timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e "$@" > $O/v_$(echo "$@" | tr ' -' '__').json 2>&1; }
run --config C3 --cycles 1000
run --config C4 --cycles 20 --no-hash-off-pass
run --config C3 --cycles 500 --lanes 2048 --no-hash-off-pass
run --config C4 --cycles 10 --lanes 4096 --no-hash-off-pass
echo done
