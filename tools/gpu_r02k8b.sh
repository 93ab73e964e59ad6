#!/bin/bash
# Kernel 8 with 8 hash accumulators: parity + C1 bench + ncu.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/k8b; mkdir -p $O
timeout 900 python -m pytest tests/test_specialize.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --kernel 8 > $O/C1_k8.json 2> $O/C1_k8.err
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --kernel 8 --no-passes > $O/C1_k8_nopass.json 2> $O/C1_k8_nopass.err
timeout 600 ncu --set full --clock-control none -k regex:rs_su -s 2 -c 1 -o $O/prof_C1_k8 -f \
   python bench.py --config C1 --steps 1 --warmup 3 --cycles 200 --no-cpu --no-e2e --no-hash-off-pass --kernel 8 > $O/ncu.log 2>&1
echo done
