#!/bin/bash
# Early register commits in kernel 7 (runtime.cu early_latch_r): kernel-7 parity (parity, edges, passes,
# waveforms, full-scope C2/C3/C4 streams), then C3 / C4 / C2 with RTLSIM_K7_EARLY_LATCH=0 (base) vs on (cur).
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/early; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_passes.py tests/test_gpu_full_scope.py -m gpu -q -p no:cacheprovider -x -k "not c5" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="--no-cpu --no-e2e --no-hash-off-pass --warmup 3"
for rep in 1 2; do
for v in base cur; do
  if [ $v = base ]; then export RTLSIM_K7_EARLY_LATCH=0; else unset RTLSIM_K7_EARLY_LATCH; fi
  for c in C3 C4 C2; do
    cyc="--cycles 1000 --steps 3"; [ $c = C4 ] && cyc="--cycles 20 --steps 2"; [ $c = C2 ] && cyc="--cycles 2000 --steps 3"
    r=$(timeout 400 python bench.py --config $c $cyc $B 2>$O/err_${v}_$c.txt | tail -1)
    echo "$rep $v $c $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); c=r["config"]; print(round(r["ms_per_step_median"]/c["cycles_per_step"]*1000,2), "us/cycle", round(r["roofline"]["frac"],4), c["launch"])' 2>&1 | tail -1)"
  done
done
done > $O/ab.txt 2>&1
echo done
