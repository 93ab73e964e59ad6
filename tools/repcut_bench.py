"""RepCut (rs_lane_opts.repcut) vs the level-synchronous single-lane kernel
(single.cuh) and its level cut (parts) on one design, single lane, CUDA-event
timed on the launching stream (hashes on device).

    python tools/repcut_bench.py [C1|C5|MC] [cycles]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_18140_b200 import rtlsim as rs  # noqa: E402
from synth import CONFIGS, config_circuit, multicore_circuit  # noqa: E402


def timed(c, n, **kw):
    g = rs.Graph(c, device=0, mode="single")
    st = torch.cuda.Stream()   # a real stream: the events must bracket the launch (not the legacy default)
    L = rs.Lanes(g, 1, stream=st, **kw)
    L.set_seed(206)
    h = torch.zeros(n, dtype=torch.uint64, device="cuda")
    L.step(n, hashes=h)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    L.step(n, hashes=h)
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / n
    out = {"us_per_cycle": round(us, 3), "shape": L.shape()}
    L.close()
    g.close()
    return out


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "MC"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    if name == "MC":
        c = multicore_circuit()
    elif name.startswith("MC"):
        k = int(name[2:])
        c = multicore_circuit(k, 200_000 // k, 60, 20_000 // k, 8, 0.01)
    else:
        c = config_circuit(name)
    gh = rs.Graph(c, device=rs.RS_DEVICE_NONE, mode="single")
    info = gh.info()
    res = {"design": name, "ops": info["n_ops"], "levels": info["n_levels"], "regs": len(c.reg_id)}
    res["level_sync"] = timed(c, n)
    for parts in (2, 4):
        if parts <= info["n_levels"]:
            res[f"level_cut{parts}"] = timed(c, n, parts=parts)
    for P in (1, 2, 4, 8, 16, 32, 64, 128, 148):
        if P > len(c.reg_id):
            continue
        st = gh.repcut_stats(P)
        r = timed(c, n, repcut=P)
        r["replication"] = round(st["ops_total"] / (info["n_ops"] + info["n_copy_ops"]), 3)
        r["max_ops"] = st["max_ops"]
        r["push"] = st["push"]
        r["kernel"] = "smem" if r["shape"]["kernel"] == 3 else "global"
        res[f"repcut{P}"] = r
        if r["kernel"] == "smem" and P in (4, 16):
            res[f"repcut{P}_global"] = timed(c, n, repcut=P, repcut_global=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
