"""Per-stage timing of the lane kernel (CTA 0) from an RS_TRACE build.

    python paper_2601_18140_b200/build.py -DRS_TRACE --out=paper_2601_18140_b200/lib/librtlsim_trace.so
    RTLSIM_LIB=paper_2601_18140_b200/lib/librtlsim_trace.so python tools/stage_trace.py C2 4

Prints, per stage type, the mean cycles spent waiting for the stage buffer
(TMA), working (slowest warp), and in the barrier.  Diagnostics only.
"""
import ctypes as C
import os
import sys
from collections import defaultdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_18140_b200 import rtlsim as rs  # noqa: E402
from synth import CONFIGS, config_circuit  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    kernel = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    lt = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    cs = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    cfg = CONFIGS[name]
    c = config_circuit(name)
    g = rs.Graph(c)
    L = rs.Lanes(g, cfg.lanes, kernel=kernel, lane_tile=lt, cluster=cs)
    L.set_seed(cfg.stim_seed)
    buf = np.zeros(4096 * 35 + 4096 * 16, dtype=np.uint64)
    L.step(2)                                     # warm
    rs._check(rs.lib().rs_debug_trace(L.h, buf.ctypes.data, buf.size))   # arm
    L.step(cycles)
    rs._check(rs.lib().rs_debug_trace(L.h, buf.ctypes.data, buf.size))
    sh = L.shape()
    nw = sh["threads"] // 32
    stride = 3 + nw
    runs = g.export("runs")
    # stage types from the host schedule are not exported; infer from count per cycle
    n = 0
    rows = []
    while n < 4096 and buf[n * stride] != 0:
        r = buf[n * stride:(n + 1) * stride].astype(np.int64)
        rows.append(r)
        n += 1
    rows = np.array(rows)
    S = len(rows) // cycles
    print(f"{name}: {len(rows)} stages traced, {S} per cycle, launch {sh}")
    wait = rows[:, 1] - rows[:, 0]
    work_max = rows[:, 3:].max(axis=1) - rows[:, 1]
    work_min = rows[:, 3:].min(axis=1) - rows[:, 1]
    bar = rows[:, 2] - rows[:, 3:].max(axis=1)
    tot = np.diff(rows[:, 0])
    print(f"per stage (cycles): total {np.mean(tot):.0f}  wait {np.mean(wait):.0f}  "
          f"work max {np.mean(work_max):.0f} min {np.mean(work_min):.0f}  barrier-after-max {np.mean(bar):.0f}")
    per_warp = (rows[:, 3:] - rows[:, 1:2]).mean(axis=0)
    print("mean work end per warp:", " ".join(f"{v:.0f}" for v in per_warp))
    ex = buf[4096 * 35:].reshape(4096, 16)[:len(rows)].astype(np.int64)
    if (ex[:, 0] != 0).all():
        print(f"extra stamp 0: {(ex[:, 0] - rows[:, 0]).mean():.0f} cycles after the loop top, "
              f"{(rows[:, 1] - ex[:, 0]).mean():.0f} before the end of the stage-buffer wait")
    for i in range(min(S, 60)):
        idx = np.arange(i, len(rows) - 1, S)
        print(f"  stage {i:3d}: total {np.mean(tot[idx]) if len(idx) else 0:8.0f} wait {np.mean(wait[idx]):7.0f} "
              f"work max {np.mean(work_max[idx]):7.0f} min {np.mean(work_min[idx]):7.0f} bar {np.mean(bar[idx]):6.0f}")


if __name__ == "__main__":
    main()
