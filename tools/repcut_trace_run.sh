#!/bin/bash
# k_repcut_smem level timing for eval variants (trace builds)
cd "$GRAFT_REPO_ROOT"
for v in ""; do
  export RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_trace$v.so
  echo "=== variant $v"
  for a in "16 0 1" "16 0 0"; do
    timeout 300 python tools/repcut_trace.py $a 2>&1 | head -3
  done
done > gpurun_out/rtrace.txt 2>&1
