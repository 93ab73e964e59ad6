#!/bin/bash
# Launch-shape sweep at the per-rank lane counts of the strong splits (C3: 2048 / 1024 / 512 lanes).
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
B="python bench.py --config C3 --cycles 500 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
run() { timeout 300 $B "$@" > $O/sw_$(echo "$@" | tr ' -' '__').json 2>&1; }
for s in "1 128 4" "1 128 2" "1 64 4" "1 64 2" "1 64 8" "2 32 2" "2 32 4" "6 64 4" "6 128 4" "6 128 2" "6 64 2"; do
  set -- $s; run --lanes 2048 --kernel $1 --lane-tile $2 --cluster $3
done
for s in "1 64 4" "1 32 4" "1 64 2" "1 128 8" "2 32 4" "2 32 2" "2 16 2" "6 64 4" "6 64 2"; do
  set -- $s; run --lanes 1024 --kernel $1 --lane-tile $2 --cluster $3
done
for s in "2 32 8" "2 16 4" "2 16 8" "2 8 4" "2 8 2" "1 32 4" "1 32 8" "1 64 8" "6 64 8"; do
  set -- $s; run --lanes 512 --kernel $1 --lane-tile $2 --cluster $3
done
echo done
