#!/bin/bash
# Kernel 7: dynamic op claiming inside the CTA (RS_K7_DYN, shared-memory counter) vs the static interleave.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/y; mkdir -p $O
DYN="RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_dyn.so RTLSIM_AUTOBUILD=0"
env $DYN timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider \
  -k "kernel7 or kernel-7 or op_pairs or c3_structure or c2_structure" > $O/pytest_dyn.log 2>&1; echo "rc=$?" >> $O/pytest_dyn.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "op_pairs or c2_structure" > $O/pytest_base.log 2>&1; echo "rc=$?" >> $O/pytest_base.log
B3="python bench.py --config C3 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
B4="python bench.py --config C4 --cycles 20 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass"
timeout 300 $B3 > $O/C3_base.json 2>&1
env $DYN timeout 300 $B3 > $O/C3_dyn.json 2>&1
timeout 300 $B4 > $O/C4_base.json 2>&1
env $DYN timeout 300 $B4 > $O/C4_dyn.json 2>&1
env $DYN timeout 300 $B3 --lanes 2048 > $O/C3_2048_dyn.json 2>&1
timeout 300 $B3 --lanes 2048 > $O/C3_2048_base.json 2>&1
timeout 300 $B3 > $O/C3_base2.json 2>&1
env $DYN timeout 300 $B3 > $O/C3_dyn2.json 2>&1

B2="python bench.py --config C2 --cycles 4000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 7 --lane-tile 32 --cluster 4"
timeout 300 $B2 --threads 896 > $O/C2_k7_t896.json 2>&1
timeout 300 $B2 --threads 1024 > $O/C2_k7_t1024.json 2>&1
env $DYN timeout 300 $B2 --threads 896 > $O/C2_k7dyn_t896.json 2>&1
env $DYN timeout 300 $B2 --threads 1024 > $O/C2_k7dyn_t1024.json 2>&1
for n in 512 256 128; do
  timeout 300 python bench.py --config C2 --lanes $n --cycles 4000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass > $O/C2_${n}_auto.json 2>&1
  timeout 300 python bench.py --config C2 --lanes $n --cycles 4000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 7 --lane-tile 32 > $O/C2_${n}_k7.json 2>&1
  env $DYN timeout 300 python bench.py --config C2 --lanes $n --cycles 4000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 7 --lane-tile 32 > $O/C2_${n}_k7dyn.json 2>&1
done
timeout 300 python bench.py --config C3 --lanes 512 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass > $O/C3_512_auto.json 2>&1
timeout 300 python bench.py --config C3 --lanes 512 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 7 > $O/C3_512_k7.json 2>&1
timeout 300 python bench.py --config C3 --lanes 1024 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass > $O/C3_1024_auto.json 2>&1
timeout 300 python bench.py --config C3 --lanes 1024 --cycles 1000 --steps 3 --warmup 3 --no-cpu --no-e2e --no-hash-off-pass --kernel 7 > $O/C3_1024_k7.json 2>&1
echo done2
