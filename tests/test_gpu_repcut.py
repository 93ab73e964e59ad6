"""GPU parity of the RepCut single-lane path (rs_lane_opts.repcut; PAPER.md
App. C, Cascade 2): P partitions (CTAs of one
cooperative launch) evaluate their registers' cones on their own state
replicas with CTA barriers only, then push register values along the Register
Update Map.  Bit-exact against the oracle: per-cycle hashes (terms summed over
the owning partitions) and the whole signal state read back from the owning
replicas."""
import numpy as np
import pytest

import oracle
from synth import CONFIGS, closed_form as cf, config_circuit, fuzz_circuit, multicore_circuit
from tests.test_gpu_parity import check, run_gpu

pytestmark = pytest.mark.gpu


GL = [0, 1, 2]   # shared-memory slices (8-byte slots when they fit) / global replicas / width-packed slices


def kernel_of(rs, c, **kw):
    g = rs.Graph(c, device=0, mode="single")
    L = rs.Lanes(g, 1, **kw)
    k = rs.lib().rs_lanes_kernel(L.h)
    L.close()
    g.close()
    return k


@pytest.mark.parametrize("gl", GL)
@pytest.mark.parametrize("P", [1, 2, 3, 8, 32])
def test_c1_repcut(rs, P, gl):
    cfg = CONFIGS["C1"]
    c = config_circuit("C1")
    assert kernel_of(rs, c, repcut=P, repcut_global=gl) == (4 if gl == 1 else 3)
    check(rs, c, cfg.cycles, 1, seed=cfg.stim_seed, mode="single", repcut=P, repcut_global=gl)


@pytest.mark.parametrize("gl", GL)
@pytest.mark.parametrize("cross_p", [0.0, 0.02, 0.3])
def test_multicore_repcut(rs, cross_p, gl):
    c = multicore_circuit(4, 500, 12, 50, 4, cross_p=cross_p, seed=9)
    for P in (1, 2, 4, 5):
        check(rs, c, 40, 1, seed=11, mode="single", repcut=P, repcut_global=gl)


@pytest.mark.parametrize("threads", [32, 64, 1024])
def test_repcut_threads(rs, threads):
    """Fewer threads than a level's ops (each thread loops over several ops,
    hash weights fetched per op) and more."""
    c = multicore_circuit(4, 2000, 12, 100, 4, cross_p=0.02, seed=4)
    check(rs, c, 25, 1, seed=8, mode="single", repcut=4, threads=threads)


@pytest.mark.parametrize("gl", GL)
def test_repcut_fuzz(rs, gl):
    for s in range(60):
        c = fuzz_circuit(8000 + s)
        R = len(c.reg_id)
        for P in sorted({1, 2, 3, 7}):
            if P <= R:
                check(rs, c, 12, 1, seed=s, mode="single", repcut=P, repcut_global=gl)


@pytest.mark.parametrize("gl", GL)
def test_repcut_closed_forms(rs, gl):
    for c in (cf.counter(16)[0], cf.lfsr(16, (16, 14, 13, 11), seed=1)[0], cf.ripple_adder(8)[0]):
        if len(c.reg_id) >= 2:
            check(rs, c, 50, 1, seed=3, mode="single", repcut=2, repcut_global=gl)


@pytest.mark.parametrize("gl", GL)
def test_repcut_chunks_and_checkpoint(rs, gl):
    """Launch boundaries, hash-off launches, staged inputs and a register
    checkpoint restore written into every replica."""
    c = multicore_circuit(3, 400, 8, 40, 4, cross_p=0.05, seed=2)
    H, F, L = run_gpu(rs, c, 30, seed=5, mode="single", repcut=3, chunks=[1, 7, 22], repcut_global=gl)
    r = oracle.simulate(c, 30, seed=5, final=True)
    assert np.array_equal(H, r.hashes)
    assert np.array_equal(F, r.final_state)
    regs = c.reg_id.tolist()
    snap = L.read(regs)
    h1 = L.step(10, hashes="host")
    L.write_registers(regs, snap)
    L.cycle = 30
    h2 = L.step(10, hashes="host")
    assert np.array_equal(h1, h2)
    L.step(5)
    h3 = L.step(3, hashes="host")
    r2 = oracle.simulate(c, 48, seed=5)
    assert np.array_equal(h3, r2.hashes[45:48])
    stim = np.random.default_rng(1).integers(0, 2**63, size=(20, len(c.input_id), 1), dtype=np.uint64)
    check(rs, c, 20, 1, mode="single", repcut=4, staged=stim, repcut_global=gl)


def test_repcut_c5(rs):
    """C5 (2M ops) does not fit shared-memory slices: the global-replica kernel."""
    cfg = CONFIGS["C5"]
    c = config_circuit("C5")
    assert kernel_of(rs, c, repcut=16) == 4
    check(rs, c, 30, 1, seed=cfg.stim_seed, mode="single", repcut=16)


def test_repcut_multicore16_smem(rs):
    """The 16-core 200k-op design of the RepCut bench: one partition per core,
    shared-memory slices; sampled parity over 20 cycles."""
    c = multicore_circuit()
    assert kernel_of(rs, c, repcut=16) == 3
    check(rs, c, 20, 1, seed=206, mode="single", repcut=16)


def test_repcut_multicore_shuffled_registers(rs):
    """Registers listed in a random order: contiguous index blocks would replicate ~10x;
    the cone clustering (compiler.cpp cone_cluster_partition) finds the cores again, so the
    16-core design still fits shared-memory slices, replication-free, and stays bit-exact."""
    import dataclasses
    c = multicore_circuit()
    perm = np.random.default_rng(3).permutation(c.n_regs)
    c = dataclasses.replace(c, reg_id=c.reg_id[perm], reg_next_id=c.reg_next_id[perm], reg_init=c.reg_init[perm])
    assert kernel_of(rs, c, repcut=16) == 3
    check(rs, c, 20, 1, seed=206, mode="single", repcut=16)
    small = multicore_circuit(n_cores=4, ops_per_core=2000, regs_per_core=200, n_levels=30, cross_p=0.05)
    perm = np.random.default_rng(4).permutation(small.n_regs)
    small = dataclasses.replace(small, reg_id=small.reg_id[perm], reg_next_id=small.reg_next_id[perm],
                                reg_init=small.reg_init[perm])
    for P, gl in [(4, 0), (4, 1), (2, 2), (8, 0)]:
        check(rs, small, 40, 1, seed=7, mode="single", repcut=P, repcut_global=gl)


def test_repcut_errors(rs):
    c = config_circuit("C1")
    g = rs.Graph(c, device=0, mode="single")
    with pytest.raises(rs.RtlSimError):
        rs.Lanes(g, 1, repcut=4, parts=2)
    with pytest.raises(rs.RtlSimError):
        rs.Lanes(g, 1, repcut=100000)
