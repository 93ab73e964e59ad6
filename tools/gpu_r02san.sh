#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over small parity runs of every step kernel.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/san; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
cat > /tmp/san_run.py <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
import oracle
from paper_2601_18140_b200 import rtlsim as rs
from synth import config_circuit, CONFIGS
from synth.edge import edge_circuit, edge_values
def chk(c, n, nl, mode="lanes", **kw):
    g = rs.Graph(c, device=0, mode=mode, passes=kw.pop("passes", False))
    L = rs.Lanes(g, nl, **kw); L.set_seed(7)
    H = L.step(n, hashes="host"); F = L.read(list(range(c.n_signals)))
    r = oracle.simulate(c, n, seed=7, n_lanes=nl, final=True)
    ok = np.array_equal(H, r.hashes) and np.array_equal(F, r.final_state)
    print(mode, kw, "ok" if ok else "MISMATCH", flush=True)
c2 = config_circuit("C2", n_ops=3000, n_levels=20, n_regs=300)
for k, lt, cs in [(7, 128, 2), (7, 32, 1), (2, 16, 2), (1, 64, 1), (6, 128, 2)]:
    chk(c2, 4, 150, kernel=k, lane_tile=lt, cluster=cs)
chk(c2, 4, 150, kernel=7, lane_tile=64, cluster=2, op_pairs=2, passes=True)
e = edge_circuit(0)
for k in (3, 5, 8):
    chk(e, 5, 1, mode="single", kernel=k)
chk(config_circuit("C1"), 20, 1, mode="single", kernel=8)
chk(config_circuit("C1"), 20, 1, mode="single", kernel=4, repcut=2)
chk(e, 3, 70, kernel=8)
PY
timeout 1200 $CS --tool memcheck --leak-check no --print-limit 20 python /tmp/san_run.py > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
timeout 1200 $CS --tool racecheck --print-limit 20 python /tmp/san_run.py > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
timeout 1200 $CS --tool synccheck --print-limit 20 python /tmp/san_run.py > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
echo done
