"""Write the cached oracle hash streams for the SURVEY.md §8(d) full parity scopes.

Calls ONLY oracle/ (and synth/ for the seeded circuit structure); nothing here
comes from the CUDA path.  The GPU tests (tests/test_gpu_full_scope.py) run
the bench's launch configuration on the GPU box and compare every sampled
(cycle, lane) hash with these files.

    python tests/golden/make_streams.py C3 C4 C5 [--threads T]

  C3  64 lanes spread over the 4,096 (first / last lane of each of the 8
      512-lane shards of §8(e)'s 8-GPU split, plus evenly spaced ones) x all
      10,000 cycles                         -> streams/C3_sampled.npz
  C4  64 lanes: 8 per 1,024-lane shard (first two, last two, four spread)
      x all 2,000 cycles                    -> streams/C4_sampled.npz
  C5  the single lane x all 100,000 cycles  -> streams/C5_full.npz
      (state carries across cycles, so no sampling is possible)

Each file holds `lanes` (global lane ids), `hashes` [cycles, lanes] (u64,
DESIGN.md reading R12), `seed`, `cycles`, the generator version tag and the
circuit's size, so a stale cache (generator changed) is detected by the test.
The C5 run is single-threaded (~19 cycles/s on the 2M-op design: ~1.5 h); it
writes a checkpoint every 5,000 cycles and resumes from it.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from synth import CONFIGS, config_circuit  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "streams")


def sample_lanes(name):
    n = CONFIGS[name].lanes
    shard = n // 8
    if name == "C3":
        s = set()
        for d in range(8):
            s |= {d * shard, d * shard + shard - 1}
        for x in np.linspace(0, n - 1, 64).astype(int).tolist():
            if len(s) >= 64:
                break
            s.add(x)
        return sorted(s)
    s = set()
    for d in range(8):
        b = d * shard
        s |= {b, b + 1, b + shard - 2, b + shard - 1}
        s |= set((b + np.linspace(0, shard - 1, 6)[1:5].astype(int)).tolist())
    return sorted(s)


def meta(name, c):
    return dict(config=name, n_ops=c.n_ops, n_signals=c.n_signals, n_regs=c.n_regs, n_inputs=c.n_inputs,
                struct_seed=CONFIGS[name].struct_seed, seed=CONFIGS[name].stim_seed)


def make_sampled(name, threads):
    c = config_circuit(name)
    cfg = CONFIGS[name]
    lanes = sample_lanes(name)
    t = time.time()
    r = oracle.simulate(c, cfg.cycles, seed=cfg.stim_seed, lanes=lanes, threads=threads)
    np.savez(os.path.join(OUT, f"{name}_sampled.npz"), lanes=np.array(lanes, dtype=np.int64),
             hashes=r.hashes, cycles=cfg.cycles, **meta(name, c))
    print(f"{name}: {len(lanes)} lanes x {cfg.cycles} cycles in {time.time() - t:.0f} s", flush=True)


def make_c5(chunk=5000):
    name = "C5"
    c = config_circuit(name)
    cfg = CONFIGS[name]
    ck = os.path.join(OUT, "C5_checkpoint.npz")
    H = np.zeros((cfg.cycles, 1), dtype=np.uint64)
    done, regs = 0, None
    if os.path.exists(ck):
        z = np.load(ck)
        done = int(z["done"])
        H[:done] = z["hashes"][:done]
        regs = z["regs"]
    t = time.time()
    while done < cfg.cycles:
        n = min(chunk, cfg.cycles - done)
        r = oracle.simulate(c, n, seed=cfg.stim_seed, cycle0=done, reg_state0=regs, final=True)
        H[done:done + n] = r.hashes
        regs = np.ascontiguousarray(r.final_state[np.asarray(c.reg_id, dtype=np.int64)])
        done += n
        np.savez(ck, done=done, hashes=H[:done], regs=regs)
        print(f"C5: {done} cycles ({time.time() - t:.0f} s)", flush=True)
    np.savez(os.path.join(OUT, "C5_full.npz"), lanes=np.array([0], dtype=np.int64), hashes=H,
             cycles=cfg.cycles, **meta(name, c))
    os.remove(ck)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 8)
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    for nm in a.names:
        if nm == "C5":
            make_c5()
        else:
            make_sampled(nm, a.threads)
