#!/bin/bash
# Kernel 7 with 16-CTA (non-portable) clusters: wide tiles on lane-poor allocations (C2 1,024 lanes: 8 tiles of
# 128 lanes x 16 CTAs = 128 SMs; C3 at 1,024 / 512 lanes).
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/z; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "op_pairs or cluster16" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B2="python bench.py --config C2 --cycles 4000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
run() { n=$1; shift; timeout 300 "$@" > $O/$n.json 2> $O/$n.err; }
run C2_k2 $B2
run C2_128x16 $B2 --kernel 7 --lane-tile 128 --cluster 16
run C2_128x16_p2 $B2 --kernel 7 --lane-tile 128 --cluster 16 --op-pairs 2
run C2_128x8 $B2 --kernel 7 --lane-tile 128 --cluster 8
run C2_64x16 $B2 --kernel 7 --lane-tile 64 --cluster 16
run C2_64x8 $B2 --kernel 7 --lane-tile 64 --cluster 8
run C2_32x16 $B2 --kernel 7 --lane-tile 32 --cluster 16
run C2_256_128x16 $B2 --lanes 256 --kernel 7 --lane-tile 128 --cluster 16
run C2_256_64x16 $B2 --lanes 256 --kernel 7 --lane-tile 64 --cluster 16
B3="python bench.py --config C3 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
run C3_1024_k2 $B3 --lanes 1024
run C3_1024_128x16 $B3 --lanes 1024 --kernel 7 --lane-tile 128 --cluster 16
run C3_1024_64x8 $B3 --lanes 1024 --kernel 7 --lane-tile 64 --cluster 8
run C3_512_k2 $B3 --lanes 512
run C3_512_128x16 $B3 --lanes 512 --kernel 7 --lane-tile 128 --cluster 16
run C3_512_64x16 $B3 --lanes 512 --kernel 7 --lane-tile 64 --cluster 16
run C3_2048_128x16 $B3 --lanes 2048 --kernel 7 --lane-tile 128 --cluster 16
run C3_2048_auto $B3 --lanes 2048
python - > $O/occ.txt 2>&1 <<'PY'
import paper_2601_18140_b200.rtlsim as rs
from synth import config_circuit
g = rs.Graph(config_circuit("C2"), device=0, passes=True)
for lt, cs, n in [(128, 16, 1024), (64, 16, 1024), (128, 16, 2048), (64, 8, 1024), (128, 8, 1024)]:
    try:
        L = rs.Lanes(g, n, kernel=7, lane_tile=lt, cluster=cs); print(lt, cs, n, L.shape())
    except Exception as e:
        print(lt, cs, n, "ERR", e)
PY
echo done
