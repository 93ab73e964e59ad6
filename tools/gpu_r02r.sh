#!/bin/bash
# C2 (1,024 lanes): kernel 7 / kernel 1 shapes vs the kernel-2 default.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
B="python bench.py --config C2 --cycles 2000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
run() { timeout 300 $B "$@" > $O/c2_$(echo "$@" | tr ' -' '__').json 2>&1; }
run --kernel 2
run --kernel 7 --lane-tile 64 --cluster 8
run --kernel 7 --lane-tile 64 --cluster 4
run --kernel 7 --lane-tile 128 --cluster 8
run --kernel 1 --lane-tile 32 --cluster 4
run --kernel 1 --lane-tile 64 --cluster 8
run --kernel 2 --lane-tile 16 --cluster 8
run --kernel 2 --lane-tile 32 --cluster 2
echo done
