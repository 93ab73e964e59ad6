"""GPU parity of the level-cut single-lane path, emulated on
one device: P partitions (CTA groups of one cooperative launch) own contiguous
level ranges and full state replicas, hand every cycle on through
release/acquire flags and push cut signals / register values into the later /
earlier replicas.  Bit-exact against the oracle: per-cycle hashes (whose
terms are summed over partitions) and the whole signal state read back from
the producing replicas."""
import numpy as np
import pytest

import oracle
from synth import CONFIGS, closed_form as cf, config_circuit, fuzz_circuit
from tests.test_gpu_parity import check, run_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("parts", [2, 3, 4, 8])
def test_c1_level_cut(rs, parts):
    cfg = CONFIGS["C1"]
    check(rs, config_circuit("C1"), cfg.cycles, 1, seed=cfg.stim_seed, mode="single", parts=parts)


def test_level_cut_fuzz(rs):
    for s in range(60):
        c = fuzz_circuit(7000 + s)
        g = rs.Graph(c, device=0, mode="single")
        nl = g.info()["n_levels"]
        g.close()
        for parts in sorted({min(2, nl), min(3, nl), min(5, nl)}):
            if parts < 2:
                continue
            check(rs, c, 12, 1, seed=s, mode="single", parts=parts)


def test_level_cut_closed_forms(rs):
    for c in (cf.counter(16)[0], cf.lfsr(16, (16, 14, 13, 11), seed=1)[0], cf.ripple_adder(8)[0]):
        g = rs.Graph(c, device=0, mode="single")
        nl = g.info()["n_levels"]
        g.close()
        if nl >= 2:
            check(rs, c, 50, 1, seed=3, mode="single", parts=2)


def test_level_cut_chunks_and_checkpoint(rs):
    """Launch boundaries (flags restart per launch), hash-off launches and a
    register checkpoint restore written into every replica."""
    c = config_circuit("C1")
    H, F, L = run_gpu(rs, c, 30, seed=5, mode="single", parts=3, chunks=[1, 7, 22])
    r = oracle.simulate(c, 30, seed=5, final=True)
    assert np.array_equal(H, r.hashes)
    regs = c.reg_id.tolist()
    snap = L.read(regs)
    h1 = L.step(10, hashes="host")
    L.write_registers(regs, snap)
    L.cycle = 30
    h2 = L.step(10, hashes="host")
    assert np.array_equal(h1, h2)
    L.step(5)                      # no hashes
    h3 = L.step(3, hashes="host")
    r2 = oracle.simulate(c, 48, seed=5)
    assert np.array_equal(h3, r2.hashes[45:48])


def test_c5_level_cut(rs):
    cfg = CONFIGS["C5"]
    c = config_circuit("C5")
    for parts in (2, 4):
        check(rs, c, 40, 1, seed=cfg.stim_seed, mode="single", parts=parts)


def test_level_cut_errors(rs):
    c = config_circuit("C1")
    g = rs.Graph(c, device=0, mode="single")
    with pytest.raises(rs.RtlSimError) as e:
        rs.Lanes(g, 1, parts=9)
    assert e.value.status == -1
    with pytest.raises(rs.RtlSimError):
        rs.Lanes(g, 1, parts=g.info()["n_levels"] + 1)
    gl = rs.Graph(c, device=0, mode="lanes")
    with pytest.raises(rs.RtlSimError):
        rs.Lanes(gl, 4, parts=2)
