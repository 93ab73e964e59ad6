#!/bin/bash
# e2e numbers (C ABI with host buffers, copies inside the timed region) for the configs the closing run timed
# device-only: C4 (100 cycles per step), C5 (5,000), C1 (default).
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/e2erest; mkdir -p $O
timeout 1500 python bench.py --config C4 --cycles 100 --steps 3 --warmup 3 --no-cpu > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 python bench.py --config C5 --cycles 5000 --steps 3 --warmup 3 --no-cpu > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu > $O/bench_C1.json 2> $O/bench_C1.err
echo done
