#!/bin/bash
# Co-resident-cluster guard: auto shapes and times across lane counts (C2 / C3 / C4 splits).
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "ragged or c3_structure or auto_kernel" > $O/pytest_t.log 2>&1; echo "pytest rc=$?" >> $O/pytest_t.log
run() { timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass "$@" > $O/t_$(echo "$@" | tr ' -' '__').json 2>&1; }
for l in 1024 512 256 128; do run --config C2 --cycles 2000 --lanes $l; done
for l in 4096 2048 1024 512; do run --config C3 --cycles 500 --lanes $l; done
for l in 8192 4096 2048 1024; do run --config C4 --cycles 10 --lanes $l; done
echo done
