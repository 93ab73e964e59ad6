#!/bin/bash
# C2 (1,024 lanes, latency-bound): kernel 2 (auto) vs kernel 7 with / without op pairs, tile and cluster shapes;
# parity of the forced-pairs kernel 7 first.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider \
  -k "op_pairs or kernel7 or kernel-7 or c2_structure" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --config C2 --cycles 4000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
run() { n=$1; shift; timeout 300 $B "$@" > $O/$n.json 2> $O/$n.err; }
run k2 
run k7_32x4_p1 --kernel 7 --lane-tile 32 --cluster 4 --op-pairs 1
run k7_32x4_p2 --kernel 7 --lane-tile 32 --cluster 4 --op-pairs 2
run k7_64x8_p1 --kernel 7 --lane-tile 64 --cluster 8 --op-pairs 1
run k7_64x8_p2 --kernel 7 --lane-tile 64 --cluster 8 --op-pairs 2
run k7_32x4_p1_t512 --kernel 7 --lane-tile 32 --cluster 4 --op-pairs 1 --threads 512
run k1_32x4 --kernel 1 --lane-tile 32 --cluster 4
run k7_64x4_p2 --kernel 7 --lane-tile 64 --cluster 4 --op-pairs 2
run k7_32x2_p2 --kernel 7 --lane-tile 32 --cluster 2 --op-pairs 2
echo done
