#!/bin/bash
cd "$GRAFT_REPO_ROOT"; export RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_trace.so
for a in "16 0 1" "16 0 0" "16 1024 1" "16 128 1" "32 0 1"; do
  timeout 300 python tools/repcut_trace.py $a
done > gpurun_out/rtrace.txt 2>&1
