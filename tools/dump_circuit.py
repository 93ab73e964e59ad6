"""Dump a config circuit for tools/slice_check.cpp: python tools/dump_circuit.py C5 /tmp/c5.bin"""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import config_circuit
c = config_circuit(sys.argv[1])
with open(sys.argv[2], "wb") as f:
    for a, dt in ((c.width, np.uint8), (c.input_id, np.uint32), (c.reg_id, np.uint32), (c.reg_next_id, np.uint32),
                  (c.reg_init, np.uint64), (c.const_id, np.uint32), (c.const_val, np.uint64), (c.opcode, np.uint8),
                  (c.out_id, np.uint32), (c.arg_off, np.uint32), (c.arg_id, np.uint32), (c.param.reshape(-1), np.uint32)):
        a = np.ascontiguousarray(a, dtype=dt)
        f.write(np.uint64(a.size).tobytes()); f.write(a.tobytes())
