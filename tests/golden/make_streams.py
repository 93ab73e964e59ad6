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

  C2  all 1,024 lanes x all 10,000 cycles (the "Full" scope): a per-cycle digest
      of every lane's hash (lane_digest below) plus 8 lanes exactly
                                            -> streams/C2_digest.npz

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


def _mix64(x):
    """splitmix64 finaliser on a uint64 array (test infrastructure: the digest below)."""
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def lane_digest(H, lanes):
    """Per-cycle digest of a [cycles, lanes] hash block: sum over lanes of
    mix64(H[c, l] + (l + 1) * golden) mod 2^64.  A wrong hash in any (cycle, lane)
    changes that cycle's digest (up to a 2^-64 collision); lanes are position-keyed."""
    with np.errstate(over="ignore"):
        key = (np.asarray(lanes, dtype=np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        return _mix64(H.astype(np.uint64) + key[None, :]).sum(axis=1, dtype=np.uint64)


def make_digest(name, threads, chunk=1000):
    c = config_circuit(name)
    cfg = CONFIGS[name]
    lanes = np.arange(cfg.lanes)
    exact = [0, 1, 2, 3, cfg.lanes - 4, cfg.lanes - 3, cfg.lanes - 2, cfg.lanes - 1]
    D = np.zeros(cfg.cycles, dtype=np.uint64)
    E = np.zeros((cfg.cycles, len(exact)), dtype=np.uint64)
    t = time.time()
    regs = None
    for c0 in range(0, cfg.cycles, chunk):  # chunks of cycles (state carried), all lanes each
        n = min(chunk, cfg.cycles - c0)
        r = oracle.simulate(c, n, seed=cfg.stim_seed, cycle0=c0, n_lanes=cfg.lanes, reg_state0=regs, final=True,
                            threads=threads)
        D[c0:c0 + n] = lane_digest(r.hashes, lanes)
        E[c0:c0 + n] = r.hashes[:, exact]
        regs = np.ascontiguousarray(r.final_state[np.asarray(c.reg_id, dtype=np.int64)])
        print(f"{name}: {c0 + n} cycles ({time.time() - t:.0f} s)", flush=True)
    np.savez(os.path.join(OUT, f"{name}_digest.npz"), digest=D, lanes=np.array(exact, dtype=np.int64), hashes=E,
             n_lanes=cfg.lanes, cycles=cfg.cycles, **meta(name, c))


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
        elif nm == "C2":
            make_digest(nm, a.threads)
        else:
            make_sampled(nm, a.threads)
