#!/bin/bash
# Kernel 8 (per-design specialised PTX): parity suite, C1 bench vs the RepCut default, launch list.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/k8; mkdir -p $O
timeout 900 python -m pytest tests/test_specialize.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-e2e > $O/C1_default.json 2> $O/C1_default.err
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-e2e --kernel 8 > $O/C1_k8.json 2> $O/C1_k8.err
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --kernel 8 > $O/C1_k8_e2e.json 2> $O/C1_k8_e2e.err
timeout 600 ncu --set full --clock-control none -k regex:rs_su -s 2 -c 1 -o $O/prof_C1_k8 -f \
   python bench.py --config C1 --steps 1 --warmup 3 --cycles 200 --no-cpu --no-e2e --no-hash-off-pass --kernel 8 > $O/ncu.log 2>&1
echo done
