"""Level timing of the single-lane kernel (CTA 0) from an RS_TRACE build.

    RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_trace.so python tools/single_trace.py C1
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_18140_b200 import rtlsim as rs  # noqa: E402
from synth import CONFIGS, config_circuit  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    c = config_circuit(name)
    g = rs.Graph(c, mode="single")
    L = rs.Lanes(g, 1, kernel=5)   # the level-synchronous grid (k_single2)
    L.set_seed(CONFIGS[name].stim_seed)
    buf = np.zeros(4096 * 35 + 4096 * 16, dtype=np.uint64)
    L.step(2, hashes="host")
    rs._check(rs.lib().rs_debug_trace(L.h, buf.ctypes.data, buf.size))  # arm
    L.step(6, hashes="host")
    rs._check(rs.lib().rs_debug_trace(L.h, buf.ctypes.data, buf.size))
    nl = g.info()["n_levels"]
    print(name, L.shape(), "levels", nl)
    for cyc in range(1, 6):
        r = buf[cyc * 64: cyc * 64 + 64].astype(np.int64)
        prev_end = buf[(cyc - 1) * 64 + 61].astype(np.int64)
        m = min(nl, 60)
        lv = np.diff(np.concatenate([[prev_end], r[:m]]))
        print(f"cycle {cyc}: levels 1..{m - 1}: mean {lv[1:].mean():.0f} min {lv[1:].min()} max {lv[1:].max()} cycles"
              f"  total {r[61] - prev_end}" + (f"  latch+inject {r[60] - r[nl - 1]}  end barrier {r[61] - r[60]}"
                                                if nl <= 60 else ""))


if __name__ == "__main__":
    main()
