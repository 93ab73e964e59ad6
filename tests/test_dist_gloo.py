"""Multi-process (world size 2, gloo, CPU) tests of the lane-sharding host
logic: shard ranges, global-lane invariance of the oracle's
results under sharding, max-over-ranks timing, per-lane result gather."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2601_18140_b200 import dist as D


def test_shards_cover_lanes_exactly():
    for world in (1, 2, 3, 4, 8):
        for total in (1, 7, 1024, 4096, 8192):
            shards = [D.shard_strong(r, world, total) for r in range(world)]
            assert shards[0].lane0 == 0
            for a, b in zip(shards, shards[1:]):
                assert a.lane0 + a.n_lanes == b.lane0
            assert sum(s.n_lanes for s in shards) == total
            assert max(s.n_lanes for s in shards) - min(s.n_lanes for s in shards) <= 1
        w = [D.shard_weak(r, world, 1024) for r in range(world)]
        assert [s.lane0 for s in w] == [1024 * r for r in range(world)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import oracle
    from synth import config_circuit
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = config_circuit("C2", n_ops=1500, n_levels=10, n_regs=150)
        sh = D.shard_strong(rank, world, 10)
        r = oracle.simulate(c, 8, seed=42, lane0=sh.lane0, n_lanes=sh.n_lanes)
        full = D.gather_lanes(r.hashes, dist)
        t = D.max_over_ranks(1.5 + rank, dist)
        q.put((rank, full, t))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_hashes_match_single_run():
    """Two ranks, each simulating its global-lane shard, reproduce one run over
    all lanes (lane ids are global), and the timing reduction is the max."""
    import oracle
    from synth import config_circuit
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = config_circuit("C2", n_ops=1500, n_levels=10, n_regs=150)
    ref = oracle.simulate(c, 8, seed=42, lane0=0, n_lanes=10).hashes
    for rank, full, t in out:
        assert np.array_equal(full, ref)
        assert t == 2.5
