#!/bin/bash
# Round-2 final GPU evidence: the whole -m gpu suite (full-scope C3 / C4 / C5 streams included), smoke,
# bench lines for every config, the ncu launch list of the default bench and one ncu --set full capture of
# its step kernel (traffic), the reference arm.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/${FINAL_DIR:-final}; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python bench.py --steps 5 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 python bench.py --config C2 --steps 5 --warmup 3 > $O/bench_C2.json 2> $O/bench_C2.err
timeout 1200 python bench.py --config C4 --cycles 100 --steps 3 --warmup 3 --no-e2e > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 python bench.py --config C5 --cycles 5000 --steps 3 --warmup 3 --no-e2e > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 python bench.py --config C1 --steps 5 --warmup 3 --no-e2e > $O/bench_C1.json 2> $O/bench_C1.err
timeout 600 python bench.py --config MC16 --repcut 16 --steps 3 --warmup 3 > $O/bench_MC16.json 2> $O/bench_MC16.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_C3.csv \
   python bench.py --steps 2 --warmup 3 --cycles 200 --no-cpu --no-e2e --no-hash-off-pass > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C3 -f \
   python bench.py --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e --no-hash-off-pass > $O/ncu_full_C3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C2 -f \
   python bench.py --config C2 --steps 1 --warmup 3 --cycles 200 --no-cpu --no-e2e --no-hash-off-pass > $O/ncu_full_C2.log 2>&1
echo done
