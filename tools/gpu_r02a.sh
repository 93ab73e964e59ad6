#!/bin/bash
# Round 2, first GPU call: the whole -m gpu suite (new edge / multi-process tests included; the
# cached full-scope streams are not written yet), the default bench line (C3), an ncu --set full
# capture of the C3 step kernel with source counters.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_full_scope.py -p no:cacheprovider \
  > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C3 -f \
   python bench.py --config C3 --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e --no-hash-off-pass > $O/ncu_full_C3.log 2>&1
echo done
