"""Lane sharding and the cross-process level cut with the product library in several
processes.

Two ranks (gloo process group, sharing this lease's one GPU -- their kernels
never wait on each other: lanes are independent) each simulate their global
lane shard [d*L/2, (d+1)*L/2) through the C ABI; the gathered per-lane hash
streams must equal a one-process run over all lanes, and the oracle on
sampled lanes.  Also: `bench.py --gpus 2` spawns its own ranks and prints one
line with n_gpus = 2 and the strong split.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LANES, CYCLES = 300, 12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _circ():
    from synth import config_circuit
    return config_circuit("C3", n_ops=20_000, n_levels=20, n_regs=2_000)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2601_18140_b200 import dist as D
    from paper_2601_18140_b200 import rtlsim as rs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        sh = D.shard_strong(rank, world, LANES)
        g = rs.Graph(_circ(), device=0)
        L = rs.Lanes(g, sh.n_lanes, lane0=sh.lane0, kernel=1 + rank)   # a different lane kernel per rank
        L.set_seed(77)
        h = L.step(CYCLES, hashes="host")
        full = D.gather_lanes(h, dist)
        q.put((rank, full, L.launches))
    finally:
        dist.destroy_process_group()


def test_two_processes_reproduce_one_process_run(rs):
    import oracle
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    c = _circ()
    g = rs.Graph(c, device=0)
    L = rs.Lanes(g, LANES)
    L.set_seed(77)
    one = L.step(CYCLES, hashes="host")
    for rank, full, launches in out:
        assert launches >= 1
        assert np.array_equal(full, one), rank
    sample = [0, LANES // 2 - 1, LANES // 2, LANES - 1]
    r = oracle.simulate(c, CYCLES, seed=77, lanes=sample, threads=4)
    assert np.array_equal(one[:, sample], r.hashes)


def test_bench_spawns_ranks():
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "C2", "--lanes", "256",
                          "--cycles", "40", "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["lanes_total"] == 256 and d["config"]["lanes_per_gpu"] == 128
    assert d["value"] > 0 and d["gpu_launches"] >= 2


def _levelcut_worker(rank, world, port, q, name, n_cycles):
    """One partition of a level cut across processes (rs_lane_opts.part_world) on this
    lease's one GPU: the ranks share the device, so they step one cycle per call in rank
    order with a host barrier between calls (their kernels never wait on each other)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2601_18140_b200 import rtlsim as rs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        c = _lc_circ(name)
        g = rs.Graph(c, device=0, mode="single")
        L = rs.Lanes(g, 1, part_world=world, part_rank=rank)
        L.set_seed(31)
        hs = [None] * world
        dist.all_gather_object(hs, L.ipc_handle())
        L.ipc_connect(hs)
        dist.barrier()
        part = np.zeros(n_cycles, dtype=np.uint64)
        for cyc in range(n_cycles):
            for r in range(world):
                if r == rank:
                    part[cyc] = L.step(1, hashes="host")[0, 0]
                    L.sync()
                dist.barrier()
        regs = L.read(c.reg_id)[:, 0]
        q.put((rank, part, regs, L.launches))
        dist.barrier()       # peers keep their memory mapped until everyone is done
    finally:
        dist.destroy_process_group()


def _lc_circ(name):
    from synth import config_circuit
    return config_circuit("C1") if name == "C1" else config_circuit("C5", n_ops=20_000, n_levels=30, n_regs=2_000)


@pytest.mark.parametrize("name,world", [("C1", 2), ("C5s", 3)])
def test_level_cut_across_processes(rs, name, world):
    """SURVEY.md §8(e) row 2 transport: partitions in separate processes reach each other's
    replicas and cycle flags through CUDA IPC mappings; the per-cycle hash is the sum of the
    partitions' shares and equals the oracle's, cycle by cycle."""
    import oracle
    port, n = _free_port(), 25
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_levelcut_worker, args=(r, world, port, q, name, n)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=900) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    H = np.zeros(n, dtype=np.uint64)
    for _, part, _, launches in out:
        H += part                                    # mod 2^64
        assert launches >= n
    c = _lc_circ(name)
    r = oracle.simulate(c, n, seed=31, final=True)
    assert np.array_equal(H, r.hashes[:, 0])
    # registers: each rank's replica holds every register's committed value
    for _, _, regs, _ in out:
        assert np.array_equal(regs, r.final_state[np.asarray(c.reg_id, dtype=np.int64), 0])
