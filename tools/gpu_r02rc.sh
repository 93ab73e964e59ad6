#!/bin/bash
# RepCut register partition by logic components: parity + MC16 / shuffled-MC16 bench.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/rc; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_repcut.py tests/test_passes.py tests/test_gpu_levelcut.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --config MC16 --repcut 16 --steps 3 --warmup 3 --no-e2e > $O/MC16.json 2> $O/MC16.err
echo done
