#!/bin/bash
# C2 (and the 4/8-GPU per-rank lane counts) on kernel 7 32-lane tiles: single ops at 1,024 threads (current)
# vs op pairs at 1,024 threads (lib/librtlsim_p1024.so, -DRS_LANES_R1_PAIRS_MAX_THREADS=1024); parity first.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/c2pairs; mkdir -p $O
RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_p1024.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider -x -k "7" > $O/pytest_p1024.log 2>&1; echo "rc=$?" >> $O/pytest_p1024.log
B="--no-cpu --no-e2e --no-hash-off-pass --warmup 3 --steps 3 --cycles 2000"
for rep in 1 2; do
for lanes in 1024 256 128; do
  r=$(python bench.py --config C2 --lanes $lanes $B 2>/dev/null | tail -1); echo "$rep cur $lanes $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); c=r["config"]; print(round(r["ms_per_step_median"]/c["cycles_per_step"]*1000,2), c["launch"])')"
  r=$(RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_p1024.so python bench.py --config C2 --lanes $lanes --op-pairs 2 $B 2>/dev/null | tail -1); echo "$rep pairs1024 $lanes $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); c=r["config"]; print(round(r["ms_per_step_median"]/c["cycles_per_step"]*1000,2), c["launch"])')"
done
done > $O/ab.txt 2>&1
echo done
