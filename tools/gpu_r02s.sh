#!/bin/bash
# Kernel 7 with 32-lane tiles (P = 1) for the lane-poor configs vs kernel 2.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "ragged or c3_structure or threads_variants" > $O/pytest_s.log 2>&1; echo "pytest rc=$?" >> $O/pytest_s.log
run() { timeout 300 python bench.py --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass "$@" > $O/s_$(echo "$@" | tr ' -' '__').json 2>&1; }
run --config C2 --kernel 7 --lane-tile 32 --cluster 4
run --config C2 --kernel 7 --lane-tile 32 --cluster 2
run --config C2 --kernel 2
run --config C3 --lanes 1024 --kernel 7 --lane-tile 32 --cluster 4
run --config C3 --lanes 1024 --kernel 2
run --config C3 --lanes 512 --kernel 7 --lane-tile 32 --cluster 4
run --config C3 --lanes 512 --kernel 7 --lane-tile 32 --cluster 8
run --config C3 --lanes 512 --kernel 2
echo done
