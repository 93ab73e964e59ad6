#!/bin/bash
# Kernel 6 with shared-atomic hash partials: parity subset, then C3 at 1024 / 768 / 512 threads.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "edges or c3_structure or ragged or wide_work or chunking or staged or checkpoint or waveform_changes or threads_variants or sharding" -p no:cacheprovider > $O/pytest_k6.log 2>&1; echo "pytest rc=$?" >> $O/pytest_k6.log
B="timeout 600 python bench.py --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
for t in 1024 768 512; do $B --kernel 6 --threads $t > $O/k6_t$t.json 2>&1; done
$B --kernel 6 --lane-tile 64 --threads 1024 > $O/k6_p2_t1024.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C3_k6 -f \
   python bench.py --kernel 6 --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e --no-hash-off-pass > $O/ncu_full_C3_k6.log 2>&1
echo done
