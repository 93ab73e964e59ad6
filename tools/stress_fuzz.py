"""Randomised parity sweep: fuzz-corpus circuits under random launch options
(lane kernel 1 / 2 / 6 / 7 / 8 or auto, tile, cluster, threads, op pairs;
single-lane kernel, RepCut partitions, level cut; graph passes on or off), hashes
and final state vs the oracle.

    python tools/stress_fuzz.py [n_cases] [seed]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2601_18140_b200 import rtlsim as rs  # noqa: E402
from synth import fuzz_circuit  # noqa: E402


def _tile(rng, kernel):
    """A lane tile valid for the lane kernel (0 = auto: let the runtime choose)."""
    if kernel == 0:
        return 0
    return int(rng.choice({1: [32, 64, 128], 7: [32, 64, 128], 6: [64, 128], 2: [8, 16, 32]}[kernel]))


def big_cases(n_cases, rng):
    """C3-shaped circuits of random size (wide-level kernel-1 paths, 4-op items,
    clusters), a few cycles, random lane counts."""
    from synth import config_circuit
    bad = 0
    for it in range(n_cases):
        n_ops = int(rng.integers(5000, 90000))
        n_levels = int(rng.integers(5, 40))
        c = config_circuit("C3", n_ops=n_ops, n_levels=n_levels, n_regs=max(1, n_ops // 10))
        kernel = int(rng.choice([1, 2, 6, 7]))
        lt = _tile(rng, kernel)
        cs = int(rng.choice([1, 2, 4]))
        nl = int(rng.integers(1, 400))
        seed = int(rng.integers(0, 1000))
        passes = bool(rng.random() < 0.5)
        g = rs.Graph(c, device=0, passes=passes)
        extra = dict(op_pairs=int(rng.integers(0, 3))) if kernel == 7 else {}
        L = rs.Lanes(g, nl, kernel=kernel, lane_tile=lt, cluster=cs, **extra)
        L.set_seed(seed)
        H = L.step(3, hashes="host")
        r = oracle.simulate(c, 3, seed=seed, n_lanes=nl, threads=8)
        ok = np.array_equal(H, r.hashes)
        bad += not ok
        print(f"big {it}: ops {n_ops} levels {n_levels} lanes {nl} kernel {kernel} lt {lt} cs {cs} passes {passes} {extra} "
              f"shape {L.shape()} -> {'ok' if ok else 'MISMATCH'}", flush=True)
        L.close()
        g.close()
    return bad


def main():
    n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 11)
    if len(sys.argv) > 3 and sys.argv[3] == "big":
        bad = big_cases(n_cases, rng)
        print("cases", n_cases, "mismatches", bad)
        sys.exit(1 if bad else 0)
    bad = 0
    for it in range(n_cases):
        seed = int(rng.integers(0, 100000))
        c = fuzz_circuit(seed)
        cycles = int(rng.integers(1, 40))
        if rng.random() < 0.6:
            mode = "lanes"
            kernel = int(rng.choice([0, 1, 2, 6, 7]))
            lt = _tile(rng, kernel)
            cs = int(rng.choice([1, 2, 4])) if kernel else 0
            nl = int(rng.integers(1, 300))
            th = int(rng.choice([0, 64, 128, 256])) if kernel else 0
            if kernel == 2 and th and th < lt:
                th = 0
            opts = dict(kernel=kernel, lane_tile=lt, cluster=cs, threads=th)
            if kernel == 7:
                opts["op_pairs"] = int(rng.integers(0, 3))
        else:
            mode, nl = "single", 1
            g0 = rs.Graph(c, device=rs.RS_DEVICE_NONE, mode="single")
            nlev, nreg = g0.info()["n_levels"], len(c.reg_id)
            g0.close()
            pick = rng.integers(0, 5)
            if pick == 0 or nreg == 0:
                opts = dict(kernel=5)
            elif pick == 1:
                opts = dict(repcut=int(rng.integers(1, min(nreg, 8) + 1)))
            elif pick == 2:
                opts = dict(repcut=int(rng.integers(1, min(nreg, 8) + 1)), repcut_global=1)
            elif pick == 3:
                opts = dict(repcut=int(rng.integers(1, min(nreg, 8) + 1)), repcut_global=2)
            else:
                opts = dict(kernel=5, parts=int(rng.integers(1, min(max(nlev, 1), 4) + 1)))
        passes = bool(rng.random() < 0.5)
        g = rs.Graph(c, device=0, mode=mode, passes=passes)
        if mode == "lanes" and rng.random() < 0.15 and len(c.reg_id):
            opts = dict(kernel=8)  # the design's own PTX (rs_specialize), lanes
        L = rs.Lanes(g, nl, **opts)
        L.set_seed(seed)
        H = L.step(cycles, hashes="host")
        F = L.read(list(range(c.n_signals)))
        r = oracle.simulate(c, cycles, seed=seed, n_lanes=nl, final=True, threads=8)
        ok = np.array_equal(H, r.hashes) and np.array_equal(F, r.final_state)
        bad += not ok
        if not ok or it % 20 == 0:
            print(f"case {it}: seed {seed} {mode} passes {passes} lanes {nl} cycles {cycles} {opts} shape {L.shape()} -> "
                  f"{'ok' if ok else 'MISMATCH'}", flush=True)
        L.close()
        g.close()
    print("cases", n_cases, "mismatches", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
