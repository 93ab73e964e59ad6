#!/bin/bash
# A/B of single-lane paths: base (lib/librtlsim_base.so) vs current
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
for rep in 1 2; do
for v in base cur; do
  if [ $v = cur ]; then unset RTLSIM_LIB; else export RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_$v.so; fi
  for c in "C5 --cycles 1000" "MC16 --repcut 16 --cycles 2000" "C5 --parts 2 --cycles 1000"; do
    r=$(timeout 400 python bench.py --config $c --steps 3 --no-cpu --no-e2e 2>/dev/null | tail -1)
    echo "$rep $v $c $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); print(round(r["ms_per_step"],3), r["clocks"]["sm_mhz"])' 2>&1 | tail -1)"
  done
done
done > $O/ab_single.txt 2>&1
