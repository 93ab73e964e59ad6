#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
export RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_trace.so
for a in "C2 4 2 32 4"; do
  echo "=== $a"; timeout 300 python tools/stage_trace.py $a 2>&1 | head -16
done > $O/trace.txt 2>&1
