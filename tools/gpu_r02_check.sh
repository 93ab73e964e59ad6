#!/bin/bash
# Re-entry check: the whole -m gpu suite, smoke and the default bench line on the current tree.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/${CHECK_DIR:-check}; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
echo done
