#!/bin/bash
# Differential exchange in the global-memory RepCut kernel (k_repcut): RepCut parity + fuzz sweep, then
# MC16 on k_repcut (P = 16) with RTLSIM_REPCUT_DIFFX=0 (full pushes) vs on.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/rcdiff; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_repcut.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python tools/stress_fuzz.py 300 41 > $O/stress.txt 2>&1; echo "rc=$?" >> $O/stress.txt
B="--no-cpu --no-e2e --no-hash-off-pass --warmup 3 --steps 3"
for rep in 1 2; do for v in off on; do
  if [ $v = off ]; then export RTLSIM_REPCUT_DIFFX=0; else unset RTLSIM_REPCUT_DIFFX; fi
  r=$(timeout 600 python bench.py --config MC16 --repcut 16 --repcut-global 1 --cycles 2000 $B 2>$O/err_$v.txt | tail -1)
  echo "$rep $v MC16 $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); c=r["config"]; print(round(r["ms_per_step_median"]/c["cycles_per_step"]*1000,2), "us/cycle", c["launch"])' 2>&1 | tail -1)"
  r=$(timeout 600 python bench.py --config C1 --repcut 4 --repcut-global 1 --kernel 0 --cycles 1000 $B 2>$O/err_c1_$v.txt | tail -1)
  echo "$rep $v C1 $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); c=r["config"]; print(round(r["ms_per_step_median"]/c["cycles_per_step"]*1000,2), "us/cycle", c["launch"])' 2>&1 | tail -1)"
done; done > $O/ab.txt 2>&1
echo done
