#!/bin/bash
# A/B of several builds on the same box (lib/librtlsim_<v>.so; "cur" = lib/librtlsim.so)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
VARIANTS=${VARIANTS:-"base cur"}
CONFIGS=${CONFIGS:-"C2 C3"}
for rep in 1 2; do
for v in $VARIANTS; do
  if [ $v = cur ]; then unset RTLSIM_LIB; else export RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_$v.so; fi
  for c in $CONFIGS; do
    cyc=""; [ $c = C3 ] && cyc="--cycles 1000"; [ $c = C4 ] && cyc="--cycles 20 --steps 2"
    r=$(timeout 400 python bench.py --config $c $cyc --steps 3 --no-cpu --no-e2e 2>/dev/null | tail -1)
    echo "$rep $v $c $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); print(r["ms_per_step"], round(r["roofline"]["frac"],4), r["clocks"]["sm_mhz"], r["config"]["launch"])' 2>&1 | tail -1)"
  done
done
done > $O/ab.txt 2>&1
