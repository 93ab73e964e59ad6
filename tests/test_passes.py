"""Graph passes of the compiler (RS_LOAD_PASSES; PAPER.md
§6.1, App. B.1): constant and copy propagation.

The oracle always runs the circuit as given; a pass is correct iff every
per-cycle hash (which covers every canonical signal, reading R12) and every
signal read back -- aliases and folded constants included -- are unchanged.
CPU tests check the pass bookkeeping through the compile-only handle; GPU
tests check results against the oracle on every kernel.
"""
import numpy as np
import pytest

import oracle
from synth import CONFIGS, config_circuit, fuzz_circuit
from synth.edge import edge_values, pass_circuit


def test_pass_bookkeeping(rs):
    for seed in range(4):
        c = pass_circuit(seed)
        g0 = rs.Graph(c, device=rs.RS_DEVICE_NONE)
        g = rs.Graph(c, device=rs.RS_DEVICE_NONE, passes=True)
        i0, i = g0.info(), g.info()
        assert i0["n_alias"] == i0["n_folded"] == 0 and i0["n_ops"] == c.n_ops
        assert i["n_ops"] + i["n_alias"] + i["n_folded"] == c.n_ops
        assert i["n_alias"] > 0 and i["n_folded"] > 0
        assert i["n_levels"] <= i0["n_levels"]
        assert i["alg_bytes_per_lane_cycle"] < i0["alg_bytes_per_lane_cycle"]
        # an alias reads its representative's row: several canonical ids share a coordinate
        sc = g.export("sig_coord")
        assert len(set(sc.tolist())) == c.n_signals - i["n_alias"]


def test_passes_on_the_c3_recipe(rs):
    """The synthetic C3 recipe has no constants, but half its signals are 1 bit wide:
    bits / shr of a 1-bit operand (lo = n = 0 by the recipe) and shifts by 0 into a
    wider result are copies, and x ^ x, x - x, eq(x, x) with both operands drawn
    equal fold to constants that then propagate."""
    c = config_circuit("C3", n_ops=30000, n_levels=20, n_regs=3000)
    i = rs.Graph(c, device=rs.RS_DEVICE_NONE, passes=True).info()
    i0 = rs.Graph(c, device=rs.RS_DEVICE_NONE).info()
    assert i["n_ops"] + i["n_alias"] + i["n_folded"] == c.n_ops
    assert 0.05 * c.n_ops < i["n_alias"] < 0.2 * c.n_ops
    assert i["alg_bytes_per_lane_cycle"] < i0["alg_bytes_per_lane_cycle"]


def test_passes_keep_repcut_replication_free(rs):
    """A multi-core design cut at its cores replicates nothing, with or without the passes:
    dead logic left by constant folding (an op of a folded constant and another core's
    register) must not be placed by that register's block (it would drag its dependents'
    cones into the other core's partition)."""
    from synth import multicore_circuit
    c = multicore_circuit()
    for passes in (False, True):
        g = rs.Graph(c, device=rs.RS_DEVICE_NONE, mode="single", passes=passes)
        i = g.info()
        st = g.repcut_stats(16)
        assert st["ops_total"] == i["n_ops"] + i["n_copy_ops"], passes
        assert st["max_ops"] <= 12_500


@pytest.mark.gpu
@pytest.mark.parametrize("mode,kernel", [("lanes", 1), ("lanes", 2), ("lanes", 6), ("lanes", 7), ("single", 3),
                                         ("single", 5)])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_gpu_passes_parity(rs, mode, kernel, seed):
    c = pass_circuit(seed)
    n = 12
    nl = 1 if mode == "single" else 70
    staged = edge_values(np.random.default_rng(seed), (n, c.n_inputs, nl))
    g = rs.Graph(c, device=0, mode=mode, passes=True)
    assert g.info()["n_alias"] > 0
    L = rs.Lanes(g, nl, stage_cycles=n, kernel=kernel)
    L.set_inputs(0, staged)
    H = np.concatenate([L.step(5, hashes="host"), L.step(n - 5, hashes="host")])
    F = L.read(list(range(c.n_signals)))
    r = oracle.simulate(c, n, n_lanes=nl, staged=staged, final=True)
    bad = np.argwhere(H != r.hashes)
    assert bad.shape[0] == 0, f"hash mismatch at (cycle, lane) {bad[:5].tolist()}"
    badf = np.argwhere(F != r.final_state)
    assert badf.shape[0] == 0, f"state mismatch at (signal, lane) {badf[:5].tolist()}"


@pytest.mark.gpu
def test_gpu_passes_fuzz_and_c3(rs):
    for seed in range(0, 60, 3):
        c = fuzz_circuit(seed)
        g = rs.Graph(c, device=0, passes=True)
        L = rs.Lanes(g, 3, kernel=(1, 2, 6)[seed % 3])
        L.set_seed(seed)
        r = oracle.simulate(c, 30, seed=seed, n_lanes=3, final=True)
        assert np.array_equal(L.step(30, hashes="host"), r.hashes), seed
        assert np.array_equal(L.read(list(range(c.n_signals))), r.final_state), seed
    c = config_circuit("C3", n_ops=30000, n_levels=20, n_regs=3000)
    hs = []
    for passes in (False, True):
        L = rs.Lanes(rs.Graph(c, device=0, passes=passes), 200, kernel=6)
        L.set_seed(CONFIGS["C3"].stim_seed)
        hs.append(L.step(8, hashes="host"))
    assert np.array_equal(hs[0], hs[1])
    r = oracle.simulate(c, 8, seed=CONFIGS["C3"].stim_seed, lanes=[0, 199], threads=2)
    assert np.array_equal(hs[1][:, [0, 199]], r.hashes)
