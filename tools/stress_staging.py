"""Stress the asynchronous staged-input path (copy stream + per-range events):
random chunk sizes and ring capacities, the next chunk staged before the
current one is stepped, hashes checked against the oracle.

    python tools/stress_staging.py [rounds]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2601_18140_b200 import rtlsim as rs  # noqa: E402
from synth import config_circuit  # noqa: E402


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rng = np.random.default_rng(7)
    circuits = {"lanes": config_circuit("C2", n_ops=3000, n_levels=15, n_regs=300), "single": config_circuit("C1")}
    bad = 0
    for it in range(rounds):
        mode = "lanes" if it % 3 else "single"
        c = circuits[mode]
        nl = int(rng.integers(1, 300)) if mode == "lanes" else 1
        ch = int(rng.integers(1, 40))
        cap = ch * int(rng.integers(2, 4)) + int(rng.integers(0, ch))
        n = ch * int(rng.integers(3, 12))
        vals = rng.integers(0, 2**63, size=(n, c.n_inputs, nl), dtype=np.int64).astype(np.uint64)
        g = rs.Graph(c, mode=mode)
        L = rs.Lanes(g, nl, stage_cycles=cap, kernel=int(rng.integers(1, 3)) if mode == "lanes" else 0)
        L.set_inputs(0, vals[0:ch])
        hs = []
        for c0 in range(0, n, ch):
            if c0 + ch < n:
                L.set_inputs(c0 + ch, vals[c0 + ch:c0 + 2 * ch])
            hs.append(L.step(ch, hashes="host"))
        H = np.concatenate(hs)
        r = oracle.simulate(c, n, n_lanes=nl, staged=vals)
        ok = np.array_equal(H, r.hashes)
        bad += not ok
        print(f"round {it}: {mode} lanes {nl} chunk {ch} ring {cap} cycles {n} -> {'ok' if ok else 'MISMATCH'}",
              flush=True)
        L.close()
        g.close()
    print("mismatches", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
