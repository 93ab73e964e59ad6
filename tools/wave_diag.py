"""Diagnostics for rs_watch on the GPU (tools/, not the product)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2601_18140_b200 import rtlsim as rs
from synth import config_circuit
c = config_circuit("C2", n_ops=3000, n_levels=15, n_regs=300)
kernel, nl, seq = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
cs = int(sys.argv[4]) if len(sys.argv) > 4 else 0
ids = [int(c.input_id[0]), int(c.reg_id[0]), 100, 200]
g = rs.Graph(c)
L = rs.Lanes(g, nl, kernel=kernel, cluster=cs)
L.set_seed(4)
for tok in seq.split(","):
    if tok == "w":
        L.watch(ids, capacity=1 << 16)
    elif tok == "h":
        L.step(1, hashes="host")
    elif tok == "n":
        L.step(1); L.sync()
    elif tok == "r":
        print("read", L.wave_read()[0].shape, flush=True)
    print("ok", tok, flush=True)
