"""SURVEY.md §8(d) parity scopes at BASELINE.json's full sizes, in the launch
configuration bench.py times, against cached oracle hash streams.

The streams (tests/golden/streams/*.npz) were written by
tests/golden/make_streams.py, which calls only oracle/ (the oracle needs
~1.5 h for C5's 100,000 single-lane cycles and ~15 min for C4's sample, too
long to recompute on every GPU run):

  C3  all 4,096 lanes x 10,000 cycles on the GPU (auto launch shape, as bench.py);
      64 sampled lanes (first / last of each 512-lane shard + 48 spread) compared
      at every cycle
  C4  the 8 lane shards of the 8-GPU split (1,024 lanes each, lane0 = d * 1,024,
      SURVEY.md §8(e)) x all 2,000 cycles, one shard at a time on this GPU;
      8 sampled lanes per shard compared at every cycle; and all 8,192 lanes in
      one allocation (the 1-GPU bench shape, kernel 7 with op pairs), 64 lanes
  C5  the single lane x all 100,000 cycles (auto single-lane kernel, as bench.py)
  C2  all 1,024 lanes x all 10,000 cycles ("Full"): a per-cycle digest of every
      lane's hash (make_streams.lane_digest) plus 8 lanes exactly, on kernel 7's
      32-lane tiles (the auto launch shape bench.py times) and on kernel 2
"""
import os

import numpy as np
import pytest

from synth import CONFIGS, config_circuit

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
STREAMS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "streams")


def _load(name, fname):
    p = os.path.join(STREAMS, fname)
    assert os.path.exists(p), f"missing {p}: run tests/golden/make_streams.py {name}"
    z = np.load(p)
    c = config_circuit(name)
    cfg = CONFIGS[name]
    # a stale cache (generator changed) must fail, not pass vacuously
    assert int(z["n_ops"]) == c.n_ops and int(z["n_signals"]) == c.n_signals
    assert int(z["struct_seed"]) == cfg.struct_seed and int(z["seed"]) == cfg.stim_seed
    return z, c, cfg


def _gpu_sampled(rs, c, seed, n_lanes, lane0, cycles, local_lanes, chunk):
    import torch
    g = rs.Graph(c, device=0, passes=True)       # bench.py's default compile (graph passes on)
    L = rs.Lanes(g, n_lanes, lane0=lane0)
    L.set_seed(seed)
    dev = torch.empty(chunk * n_lanes, dtype=torch.int64, device="cuda")
    idx = torch.as_tensor(local_lanes, dtype=torch.int64, device="cuda")
    out = np.zeros((cycles, len(local_lanes)), dtype=np.uint64)
    done = 0
    while done < cycles:
        n = min(chunk, cycles - done)
        L.step(n, hashes=dev[:n * n_lanes])
        L.sync()
        out[done:done + n] = dev[:n * n_lanes].view(n, n_lanes)[:, idx].cpu().numpy().view(np.uint64)
        done += n
    shape = L.shape()
    L.close()
    g.close()
    return out, shape


def test_c3_full_cycles_sampled_lanes(rs):
    z, c, cfg = _load("C3", "C3_sampled.npz")
    lanes = [int(x) for x in z["lanes"]]
    H, shape = _gpu_sampled(rs, c, cfg.stim_seed, cfg.lanes, 0, cfg.cycles, lanes, 1000)
    bad = np.argwhere(H != z["hashes"])
    assert bad.shape[0] == 0, f"C3 {shape}: mismatch at (cycle, sample) {bad[:5].tolist()}"


def test_c4_shards_full_cycles_sampled_lanes(rs):
    z, c, cfg = _load("C4", "C4_sampled.npz")
    lanes = np.asarray(z["lanes"], dtype=np.int64)
    shard = cfg.lanes // 8
    for d in range(8):
        sel = np.nonzero((lanes >= d * shard) & (lanes < (d + 1) * shard))[0]
        assert sel.size >= 8
        H, shape = _gpu_sampled(rs, c, cfg.stim_seed, shard, d * shard, cfg.cycles,
                                (lanes[sel] - d * shard).tolist(), 250)
        bad = np.argwhere(H != z["hashes"][:, sel])
        assert bad.shape[0] == 0, f"C4 shard {d} {shape}: mismatch at (cycle, sample) {bad[:5].tolist()}"


def test_c4_bench_shape_full_cycles_sampled_lanes(rs):
    """C4 as bench.py times it on one GPU: all 8,192 lanes in one allocation (auto: kernel 7 with op
    pairs), graph passes on, all 2,000 cycles; the 64 cached lanes (spread over the 8 shards) compared
    at every cycle."""
    z, c, cfg = _load("C4", "C4_sampled.npz")
    lanes = [int(x) for x in z["lanes"]]
    H, shape = _gpu_sampled(rs, c, cfg.stim_seed, cfg.lanes, 0, cfg.cycles, lanes, 250)
    assert shape["kernel"] == 7
    bad = np.argwhere(H != z["hashes"])
    assert bad.shape[0] == 0, f"C4 {shape}: mismatch at (cycle, sample) {bad[:5].tolist()}"


def test_c5_all_100k_cycles(rs):
    z, c, cfg = _load("C5", "C5_full.npz")
    g = rs.Graph(c, device=0, mode="single", passes=True)
    L = rs.Lanes(g, 1)
    L.set_seed(cfg.stim_seed)
    H = np.concatenate([L.step(20_000, hashes="host") for _ in range(cfg.cycles // 20_000)])
    bad = np.argwhere(H != z["hashes"])
    assert bad.shape[0] == 0, f"C5 {L.shape()}: mismatch at cycles {bad[:5, 0].tolist()}"


@pytest.mark.parametrize("kernel", [2, 7])
def test_c2_all_lanes_all_cycles(rs, kernel):
    import torch
    from tests.golden.make_streams import lane_digest
    z, c, cfg = _load("C2", "C2_digest.npz")
    g = rs.Graph(c, device=0, passes=True)
    L = rs.Lanes(g, cfg.lanes, kernel=kernel, lane_tile=32)
    L.set_seed(cfg.stim_seed)
    n_l, chunk = cfg.lanes, 1000
    dev = torch.empty(chunk * n_l, dtype=torch.int64, device="cuda")
    lanes = np.arange(n_l)
    exact = np.asarray(z["lanes"], dtype=np.int64)
    for c0 in range(0, cfg.cycles, chunk):
        n = min(chunk, cfg.cycles - c0)
        L.step(n, hashes=dev[:n * n_l])
        L.sync()
        H = dev[:n * n_l].view(n, n_l).cpu().numpy().view(np.uint64)
        bad = np.nonzero(lane_digest(H, lanes) != z["digest"][c0:c0 + n])[0]
        assert bad.size == 0, f"C2 {L.shape()}: digest mismatch at cycles {(bad[:5] + c0).tolist()}"
        assert np.array_equal(H[:, exact], z["hashes"][c0:c0 + n]), f"C2 {L.shape()}: exact lanes differ"
    L.close()
    g.close()
