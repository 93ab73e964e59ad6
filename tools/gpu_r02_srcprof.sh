#!/bin/bash
# Source-level (SASS) profile of the headline kernel (kernel 7 on C3) and of C2's kernel 2:
# per-instruction executed counts and stall samples, read here with ncu -i --page source.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/srcprof; mkdir -p $O
python bench.py --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e --no-hash-off-pass > $O/plain_C3.json 2> $O/plain_C3.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C3 -f \
   python bench.py --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e --no-hash-off-pass > $O/ncu_C3.log 2>&1
python bench.py --config C2 --steps 1 --warmup 3 --cycles 200 --no-cpu --no-e2e --no-hash-off-pass > $O/plain_C2.json 2> $O/plain_C2.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C2 -f \
   python bench.py --config C2 --steps 1 --warmup 3 --cycles 200 --no-cpu --no-e2e --no-hash-off-pass > $O/ncu_C2.log 2>&1
echo done
