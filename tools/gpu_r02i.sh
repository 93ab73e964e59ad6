#!/bin/bash
# Per-rank lane counts of the 2/4/8-GPU strong splits, measured on one GPU (predicts the scaling curve);
# plus the caller-owned-state test.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -k "caller_owned or l2_policy" -m gpu -q -p no:cacheprovider > $O/pytest_i.log 2>&1; echo "pytest rc=$?" >> $O/pytest_i.log
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
for l in 4096 2048 1024 512; do timeout 600 $B --config C3 --cycles 1000 --lanes $l > $O/split_C3_$l.json 2>&1; done
for l in 8192 4096 2048 1024; do timeout 900 $B --config C4 --cycles 20 --lanes $l > $O/split_C4_$l.json 2>&1; done
for l in 1024 512 256 128; do timeout 600 $B --config C2 --cycles 2000 --lanes $l > $O/split_C2_$l.json 2>&1; done
echo done
