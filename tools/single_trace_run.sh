cd "$GRAFT_REPO_ROOT"; export RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_trace.so
timeout 300 python tools/single_trace.py C1 > gpurun_out/strace.txt 2>&1
timeout 300 python tools/single_trace.py C5 >> gpurun_out/strace.txt 2>&1
