#!/bin/bash
# Full GPU suite (graph passes, kernel 6, full-scope C3/C4 streams), default bench line, kernel-6 bench.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_full_scope.py::test_c5_all_100k_cycles \
  --durations=15 > $O/pytest_gpu_f.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_f.log
timeout 1200 python bench.py --steps 3 --warmup 3 > $O/bench_C3_f.json 2> $O/bench_C3_f.err
timeout 600 python bench.py --kernel 6 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_k6_f.json 2> $O/bench_C3_k6_f.err
timeout 600 python bench.py --kernel 1 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-passes > $O/bench_C3_k1_nopass.json 2> $O/bench_C3_k1_nopass.err
echo done
