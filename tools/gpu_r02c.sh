#!/bin/bash
# Kernel 6 A/B: L1 prefetch of the next work item's operand rows (default build) vs none.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "edges_lanes or c3_structure or ragged or wide_work" -p no:cacheprovider > $O/pytest_k6.log 2>&1; echo "pytest rc=$?" >> $O/pytest_k6.log
for v in pf nopf; do
  L=""; [ $v = nopf ] && L="RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_nopf.so RTLSIM_AUTOBUILD=0"
  for k in 6 1; do
    env $L timeout 600 python bench.py --kernel $k --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass > $O/bench_C3_k${k}_$v.json 2> $O/bench_C3_k${k}_$v.err
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C3_k6 -f \
   python bench.py --kernel 6 --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e --no-hash-off-pass > $O/ncu_full_C3_k6.log 2>&1
echo done
