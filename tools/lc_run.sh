python -m pytest tests/test_gpu_levelcut.py -x -q 2>&1 | tail -3
python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
for p in 0 2 4; do python bench.py --config C5 --cycles 2000 --steps 3 --warmup 3 --no-e2e --no-cpu --parts $p 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('C5 parts', $p, d['ms_per_step']/2000*1e3, 'us/cycle', d['config']['launch'])"; done
for p in 0 2 4; do python bench.py --config C1 --cycles 20000 --steps 3 --warmup 3 --no-e2e --no-cpu --parts $p 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('C1 parts', $p, d['ms_per_step']/20000*1e3, 'us/cycle', d['config']['launch'])"; done
