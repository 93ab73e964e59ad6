#!/bin/bash
# Kernel 8 multi-warp single lane: parity + C1 per warp count.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/k8c; mkdir -p $O
timeout 900 python -m pytest tests/test_specialize.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for W in 1 2 3 4 5 6 8; do
  RTLSIM_K8_WARPS=$W timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-e2e --no-cpu --kernel 8 > $O/C1_w$W.json 2> $O/C1_w$W.err
done
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --kernel 8 > $O/C1_auto.json 2> $O/C1_auto.err
echo done
