#!/bin/bash
# Cross-process level cut (lockstep on one GPU), graph-pass parity, kernel-6 + passes bench.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_passes.py tests/test_gpu_levelcut.py -m gpu -q -p no:cacheprovider > $O/pytest_g.log 2>&1; echo "pytest rc=$?" >> $O/pytest_g.log
timeout 600 python bench.py --kernel 6 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_C3_k6_g.json 2> $O/bench_C3_k6_g.err
echo done
