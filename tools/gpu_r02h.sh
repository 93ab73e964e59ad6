#!/bin/bash
# L2-residency policy A/B (C2, C3, C4) + its parity test.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -k l2_policy -m gpu -q -p no:cacheprovider > $O/pytest_h.log 2>&1; echo "pytest rc=$?" >> $O/pytest_h.log
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
for p in 0 1 2; do
  timeout 600 $B --config C2 --cycles 2000 --l2-policy $p > $O/l2_C2_p$p.json 2>&1
  timeout 600 $B --config C3 --cycles 1000 --l2-policy $p > $O/l2_C3_p$p.json 2>&1
  timeout 900 $B --config C4 --cycles 20 --l2-policy $p > $O/l2_C4_p$p.json 2>&1
done
echo done
