#!/bin/bash
# Full GPU validation + bench lines + profiles (one gpurun call).
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
timeout 900 python bench.py --config C3 --cycles 1000 --steps 3 > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 python bench.py --config C4 --cycles 20 --steps 2 --warmup 3 --no-e2e > $O/bench_C4.json 2> $O/bench_C4.err
timeout 600 python bench.py --config C5 --cycles 2000 --steps 3 --no-e2e > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 python bench.py --config C1 --cycles 1000 --steps 3 --no-e2e > $O/bench_C1.json 2> $O/bench_C1.err
timeout 600 python bench.py --config MC16 --repcut 16 --cycles 2000 --steps 3 > $O/bench_MC16_repcut16.json 2> $O/bench_MC16.err
timeout 600 python bench.py --config C1 --repcut 2 --cycles 2000 --steps 3 --no-e2e > $O/bench_C1_repcut2.json 2> $O/bench_C1_repcut.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_C2.csv \
   python bench.py --steps 2 --warmup 3 --cycles 1000 --no-cpu > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C2 -f \
   python bench.py --steps 1 --warmup 3 --cycles 200 --no-cpu --no-e2e > $O/ncu_full_C2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanes -s 3 -c 1 -o $O/prof_C3 -f \
   python bench.py --config C3 --steps 1 --warmup 3 --cycles 20 --no-cpu --no-e2e > $O/ncu_full_C3.log 2>&1
bash tools/ncu_repcut.sh
echo done
