"""Full-scope parity at BASELINE.json sizes (SURVEY.md §8(d) "Parity scope"),
in the bench's launch configuration: the GPU runs every lane for every cycle
(hashes on the device), the oracle recomputes the prescribed lane sample
cycle by cycle, and every (cycle, lane) hash must match.

    python tools/full_parity.py [C2|C3|C4|C5 ...]

  C2  all 1,024 lanes x 10,000 cycles
  C3  64 evenly spaced lanes (incl. first / last of each 128-lane tile group)
      x 10,000 cycles, plus all 4,096 lanes for the first 100 cycles
  C4  ~32 lanes spread over the 8 would-be GPU shards (first / last lane of
      each) x 400 cycles, plus 128 lanes for the first 10 cycles (the oracle
      needs ~0.15 s per lane-cycle of the 2M-op design)
  C5  the single lane x C5_CYCLES (default 10,000; the single-threaded oracle
      is the limit) cycles, plus the final state
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2601_18140_b200 import rtlsim as rs  # noqa: E402
from synth import CONFIGS, config_circuit  # noqa: E402

THREADS = os.cpu_count() or 8


def gpu_hashes(c, mode, lanes, cycles, seed, chunk):
    g = rs.Graph(c, device=0, mode=mode)
    L = rs.Lanes(g, lanes)
    L.set_seed(seed)
    H = np.zeros((cycles, lanes), dtype=np.uint64)
    dev = torch.empty(chunk * lanes, dtype=torch.int64, device="cuda")
    done = 0
    while done < cycles:
        n = min(chunk, cycles - done)
        L.step(n, hashes=dev[:n * lanes])
        torch.cuda.synchronize()  # the library's own stream is not ordered with torch's
        H[done:done + n] = dev[:n * lanes].view(n, lanes).cpu().numpy().view(np.uint64)
        done += n
    F = L.read(list(range(c.n_signals))) if mode == "single" else None
    shape = L.shape()
    L.close()
    g.close()
    return H, F, shape


def check(name):
    cfg = CONFIGS[name]
    c = config_circuit(name)
    t0 = time.time()
    res = {"config": name}
    if name == "C2":
        H, _, shape = gpu_hashes(c, "lanes", 1024, 10000, cfg.stim_seed, 1000)
        r = oracle.simulate(c, 10000, seed=cfg.stim_seed, n_lanes=1024, threads=THREADS)
        res.update(scope="all 1024 lanes x 10000 cycles", ok=bool(np.array_equal(H, r.hashes)))
    elif name in ("C3", "C4"):
        lanes, cycles, head_cycles, head_lanes = (4096, 10000, 100, 4096) if name == "C3" else (8192, 400, 10, 128)
        H, _, shape = gpu_hashes(c, "lanes", lanes, cycles, cfg.stim_seed, 100 if name == "C3" else 10)
        shard = lanes // 8
        n_spread = 48 if name == "C3" else 16
        sample = sorted(set(list(np.linspace(0, lanes - 1, n_spread).astype(int)) +
                            [k * shard for k in range(8)] + [k * shard + shard - 1 for k in range(8)]))
        r = oracle.simulate(c, cycles, seed=cfg.stim_seed, lanes=sample, threads=THREADS)
        ok1 = bool(np.array_equal(H[:, sample], r.hashes))
        r2 = oracle.simulate(c, head_cycles, seed=cfg.stim_seed, n_lanes=head_lanes, threads=THREADS)
        ok2 = bool(np.array_equal(H[:head_cycles, :head_lanes], r2.hashes))
        res.update(scope=f"{len(sample)} lanes x {cycles} cycles + {head_lanes} lanes x {head_cycles} cycles",
                   ok=ok1 and ok2, sampled_ok=ok1, head_ok=ok2)
    else:  # C5
        n = int(os.environ.get("C5_CYCLES", "10000"))
        H, F, shape = gpu_hashes(c, "single", 1, n, cfg.stim_seed, min(n, 10000))
        r = oracle.simulate(c, n, seed=cfg.stim_seed, final=True, threads=1)
        res.update(scope=f"1 lane x {n} cycles + final state",
                   ok=bool(np.array_equal(H, r.hashes) and np.array_equal(F, r.final_state)))
    res.update(launch=shape, seconds=round(time.time() - t0, 1), oracle_threads=THREADS)
    print(json.dumps(res), flush=True)
    return res["ok"]


if __name__ == "__main__":
    names = sys.argv[1:] or ["C2", "C3", "C5", "C4"]
    ok = all([check(n) for n in names])
    sys.exit(0 if ok else 1)
