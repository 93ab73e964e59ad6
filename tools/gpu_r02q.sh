#!/bin/bash
# After the RepCut dead-logic placement fix: RepCut / passes / level-cut tests, MC16 bench (passes on / off).
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_repcut.py tests/test_passes.py tests/test_gpu_levelcut.py -m gpu -q -p no:cacheprovider > $O/pytest_q.log 2>&1; echo "pytest rc=$?" >> $O/pytest_q.log
timeout 600 python bench.py --config MC16 --repcut 16 --steps 3 --warmup 3 > $O/q_MC16.json 2> $O/q_MC16.err
timeout 600 python bench.py --config MC16 --repcut 16 --steps 3 --warmup 3 --no-passes --no-cpu --no-e2e > $O/q_MC16_nopass.json 2> $O/q_MC16_nopass.err
echo done
