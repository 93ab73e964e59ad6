#!/bin/bash
# Level cut with differential register exchange: single-device level-cut, cross-process and RepCut
# parity; C2 on kernel 2 (auto) vs kernel 7 at 32-lane tiles / 1,024 threads.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/diffx; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_levelcut.py tests/test_gpu_multiproc.py tests/test_gpu_repcut.py tests/test_gpu_full_scope.py::test_c5_all_100k_cycles -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for rep in 1 2; do
  python bench.py --config C2 --cycles 2000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass > $O/c2_auto_$rep.json 2>/dev/null
  python bench.py --config C2 --cycles 2000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 7 --lane-tile 32 --threads 1024 > $O/c2_k7_$rep.json 2>/dev/null
  python bench.py --config C5 --cycles 2000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --parts 2 > $O/c5_p2_$rep.json 2>/dev/null
done
echo done
