#!/bin/bash
# ncu --set full captures of the other configs' step kernels (C4 kernel 7 with op pairs, C5 level-synchronous
# grid, MC16 RepCut) for their traffic files and summaries; each command first runs plain (exit 0) then under ncu.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/ncurest; mkdir -p $O
B="--no-cpu --no-e2e --no-hash-off-pass"
python bench.py --config C4 --cycles 2 --steps 1 --warmup 3 $B > $O/plain_C4.json 2>$O/plain_C4.err && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C4 -f \
   python bench.py --config C4 --cycles 2 --steps 1 --warmup 3 $B > $O/ncu_C4.log 2>&1
python bench.py --config C5 --cycles 200 --steps 1 --warmup 3 $B > $O/plain_C5.json 2>$O/plain_C5.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_single -s 3 -c 1 -o $O/prof_C5 -f \
   python bench.py --config C5 --cycles 200 --steps 1 --warmup 3 $B > $O/ncu_C5.log 2>&1
python bench.py --config MC16 --repcut 16 --cycles 2000 --steps 1 --warmup 3 $B > $O/plain_MC16.json 2>$O/plain_MC16.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_repcut -s 3 -c 1 -o $O/prof_MC16 -f \
   python bench.py --config MC16 --repcut 16 --cycles 2000 --steps 1 --warmup 3 $B > $O/ncu_MC16.log 2>&1
echo done
