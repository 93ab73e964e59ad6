#!/bin/bash
# A/B of kernel-7 variants on one box: "base" = lib/librtlsim_base.so (built -DRS_NO_L2PF
# -DRS_K7_LATCH_U=2: the round's committed kernel 7), "nopf" = the current library with
# RTLSIM_K7_PREFETCH=0, "cur" = the current library.  Kernel-7 parity tests first.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/${AB_DIR:-ab2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
VARIANTS=${VARIANTS:-"base nopf cur"}
CONFIGS=${CONFIGS:-"C3 C4"}
for rep in 1 2; do
for v in $VARIANTS; do
  unset RTLSIM_LIB RTLSIM_K7_PREFETCH
  case $v in base) export RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_base.so;; nopf) export RTLSIM_K7_PREFETCH=0;; esac
  for c in $CONFIGS; do
    cyc="--cycles 1000 --steps 3"; [ $c = C4 ] && cyc="--cycles 20 --steps 2"
    r=$(timeout 400 python bench.py --config $c $cyc --warmup 3 --no-cpu --no-e2e --no-hash-off-pass 2>$O/err_${v}_$c.txt | tail -1)
    echo "$rep $v $c $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); print(r["ms_per_step_median"], round(r["roofline"]["frac"],4), r["clocks"]["sm_mhz"], r["config"]["launch"])' 2>&1 | tail -1)"
  done
done
done > $O/ab.txt 2>&1
echo done
