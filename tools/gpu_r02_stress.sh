#!/bin/bash
# Randomised parity sweeps on the final tree (tools/stress_fuzz.py): fuzz-corpus circuits under random
# launch options (every lane kernel incl. 7 / 8 and auto, op pairs, passes; single-lane kernels, RepCut,
# level cut), and C3-shaped circuits of random size on kernels 1 / 2 / 6 / 7.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/stress; mkdir -p $O
timeout 1500 python tools/stress_fuzz.py 600 23 > $O/stress_fuzz.txt 2>&1; echo "rc=$?" >> $O/stress_fuzz.txt
timeout 1200 python tools/stress_fuzz.py 60 29 big > $O/stress_big.txt 2>&1; echo "rc=$?" >> $O/stress_big.txt
echo done
