#!/bin/bash
# Per-rank lane counts of the 2/4/8-GPU strong splits on one B200 (the final tree, auto launch shapes).
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/split_final; mkdir -p $O
B="--no-cpu --no-e2e --no-hash-off-pass --warmup 3"
run() { local n=$1; shift; r=$(timeout 600 python bench.py "$@" $B 2>$O/$n.err | tail -1); echo "$r" > $O/$n.json
  echo "$n $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); c=r["config"]; print(round(r["ms_per_step_median"]/c["cycles_per_step"]*1000,2), "us/cycle", c["launch"])' 2>&1 | tail -1)"; }
{
for l in 2048 1024 512; do run C3_$l --config C3 --lanes $l --cycles 1000 --steps 3; done
for l in 4096 2048 1024; do run C4_$l --config C4 --lanes $l --cycles 20 --steps 2; done
for l in 512 256 128; do run C2_$l --config C2 --lanes $l --cycles 2000 --steps 3; done
} > $O/split.txt 2>&1
echo done
