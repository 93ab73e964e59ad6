#!/bin/bash
# Kernel 2 vs kernel 7 below 2,048 lanes (the auto rule's threshold): per-rank lane counts of the
# 2/4/8-GPU strong splits (C2 1,024..128; C3 1,024 / 512; C4 1,024).
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/k7low; mkdir -p $O
run() { # name args...
  local n=$1; shift
  r=$(timeout 400 python bench.py "$@" --warmup 3 --no-cpu --no-e2e --no-hash-off-pass 2>$O/$n.err | tail -1)
  echo "$n $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); c=r["config"]; print(round(r["ms_per_step_median"]/c["cycles_per_step"]*1000,2), "us/cycle", c["launch"])' 2>&1 | tail -1)"
}
for k in 2 7; do
  run C2_1024_k$k --config C2 --cycles 2000 --steps 3 --kernel $k
  run C2_512_k$k --config C2 --lanes 512 --cycles 2000 --steps 3 --kernel $k
  run C2_256_k$k --config C2 --lanes 256 --cycles 2000 --steps 3 --kernel $k
  run C2_128_k$k --config C2 --lanes 128 --cycles 2000 --steps 3 --kernel $k
  run C3_1024_k$k --config C3 --lanes 1024 --cycles 500 --steps 3 --kernel $k
  run C3_512_k$k --config C3 --lanes 512 --cycles 500 --steps 3 --kernel $k
  run C4_1024_k$k --config C4 --lanes 1024 --cycles 20 --steps 2 --kernel $k
done > $O/k7low.txt 2>&1
echo done
