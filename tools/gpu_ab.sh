#!/bin/bash
# Kernel-7 parity tests on the current library, then an A/B of library builds
# (VARIANTS: "cur" = lib/librtlsim.so, X = lib/librtlsim_X.so) on CONFIGS.  Output: gpurun_out/$AB_DIR.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/${AB_DIR:-ab}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
VARIANTS=${VARIANTS:-"base cur"}
CONFIGS=${CONFIGS:-"C3 C4"}
for rep in 1 2; do
for v in $VARIANTS; do
  if [ $v = cur ]; then unset RTLSIM_LIB; else export RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_$v.so; fi
  for c in $CONFIGS; do
    cyc="--cycles 1000 --steps 3"; [ $c = C4 ] && cyc="--cycles 20 --steps 2"; [ $c = C2 ] && cyc="--cycles 2000 --steps 3"
    r=$(timeout 400 python bench.py --config $c $cyc --warmup 3 --no-cpu --no-e2e --no-hash-off-pass 2>$O/err_${v}_$c.txt | tail -1)
    echo "$rep $v $c $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); print(r["ms_per_step_median"], round(r["roofline"]["frac"],4), r["clocks"]["sm_mhz"], r["config"]["launch"])' 2>&1 | tail -1)"
  done
done
done > $O/ab.txt 2>&1
echo done
