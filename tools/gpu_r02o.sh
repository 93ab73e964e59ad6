#!/bin/bash
# Kernel 7 adaptive pairs: parity (wide items = pairs on), C3 / C4 benches.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_passes.py -m gpu -q -x -p no:cacheprovider \
  -k "kernel7 or kernel-7 or 7 or c3_structure or fuzz_corpus or wide_work or auto_kernel" > $O/pytest_o.log 2>&1; echo "pytest rc=$?" >> $O/pytest_o.log
timeout 600 python bench.py --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/o_C3.json 2>&1
timeout 900 python bench.py --config C4 --cycles 20 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass > $O/o_C4.json 2>&1
timeout 900 python bench.py --config C4 --cycles 20 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --lanes 2048 > $O/o_C4_2048.json 2>&1
echo done
