"""Per-level timing of k_repcut_smem (partition 0) from an RS_TRACE build.

    RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_trace.so python tools/repcut_trace.py [P] [threads] [hash]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_18140_b200 import rtlsim as rs  # noqa: E402
from synth import multicore_circuit  # noqa: E402


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    th = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    hashes = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
    c = multicore_circuit()
    g = rs.Graph(c, device=0, mode="single")
    L = rs.Lanes(g, 1, repcut=P, threads=th)
    L.set_seed(206)
    buf = np.zeros(4096 * 35 + 4096 * 16, dtype=np.uint64)
    hd = torch.zeros(8, dtype=torch.uint64, device="cuda")
    L.step(2, hashes=hd if hashes else None)
    rs._check(rs.lib().rs_debug_trace(L.h, buf.ctypes.data, buf.size))  # arm
    L.step(6, hashes=hd if hashes else None)
    rs._check(rs.lib().rs_debug_trace(L.h, buf.ctypes.data, buf.size))
    nl = g.info()["n_levels"]
    print("P", P, L.shape(), "levels", nl, "hash", hashes)
    for cyc in range(1, 6):
        r = buf[cyc * 64: cyc * 64 + 64].astype(np.int64)
        prev_end = buf[(cyc - 1) * 64 + 62].astype(np.int64)
        lv = np.diff(np.concatenate([[prev_end], r[:nl]]))
        print(f"cycle {cyc}: inject+L0 {lv[0]} levels mean {lv[1:].mean():.0f} min {lv[1:].min()} max {lv[1:].max()}"
              f"  commit+hash {r[60] - r[nl - 1]}  grid barrier {r[61] - r[60]}  pull {r[62] - r[61]}"
              f"  total {r[62] - prev_end}")


if __name__ == "__main__":
    main()
