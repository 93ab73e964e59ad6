#!/bin/bash
# ncu --set full of k_repcut_smem on the 16-core design (P = 16)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
cat > /tmp/rc_run.py <<'PY'
import sys
sys.path.insert(0, ".")
import torch
from paper_2601_18140_b200 import rtlsim as rs
from synth import multicore_circuit
c = multicore_circuit()
g = rs.Graph(c, device=0, mode="single")
L = rs.Lanes(g, 1, repcut=16)
L.set_seed(206)
h = torch.zeros(200, dtype=torch.uint64, device="cuda")
for _ in range(4):
    L.step(200, hashes=h)
torch.cuda.synchronize()
print("ok")
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_repcut_smem -s 2 -c 1 -o $O/prof_repcut -f \
   python /tmp/rc_run.py > $O/ncu_repcut.log 2>&1
