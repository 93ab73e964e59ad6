import sys, traceback
sys.path.insert(0, '.')
import numpy as np
from paper_2601_18140_b200 import rtlsim as rs
from synth import Builder
def run(c, n, lanes, mode='lanes'):
    try:
        g = rs.Graph(c, mode=mode); L = rs.Lanes(g, lanes); L.set_seed(1); h = L.step(n, hashes='host'); print('ok', h.shape)
    except Exception as e:
        print('FAIL', e)
b = Builder(); r = b.reg(8, 3); b.set_next(r, r); run(b.build(), 5, 3)
b = Builder(); b.input(12); b.input(64); run(b.build(), 5, 70)
b = Builder(); k = b.const(64, 2**64-1); k2 = b.const(7, 5); b.op('add', [k, k2], 64); b.op('cat', [k2, k], 64)
c = b.build(); run(c, 3, 1); run(c, 3, 1, 'single')
