"""Op-semantics edge cases through rs_step_cycles on every step kernel.

The circuit (synth.edge.edge_circuit) puts each op of the vocabulary at the
corners of its semantics -- shl / shr by 0, 1, w-1, w, 63, 64, 65, 4096;
not into a wider out width (reading R3); bits with hi = 63; cat with
w_b = 1 / 63 / 64; mux with 2..64-bit selectors; and/or/xor/add/sub/mul folds
of 4..8 and 63 operands -- and the staged inputs are biased to 0, all ones,
1, 2^63 and sparse bits (synth.edge.edge_values), one (cycle, lane) per
value.  The oracle is pinned on this very circuit against the big-integer
definitions (tests/bigint_ref.py, CPU test below); the GPU tests compare
per-cycle hashes and the full final state with the oracle bit for bit, on
lane kernel 1 (P = 1, 2, 4; cluster 1 and 2), lane kernel 2 (8/16/32-lane
tiles), and the single-lane kernels 3 (RepCut, shared memory; P = 1, 2),
4 (RepCut, global replicas), 5 (level-synchronous grid) and the level cut.
"""
import numpy as np
import pytest

import oracle
from synth.edge import edge_circuit, edge_values

from . import bigint_ref as R


def _staged(c, cycles, lanes, seed):
    return edge_values(np.random.default_rng(seed), (cycles, c.n_inputs, lanes))


@pytest.mark.parametrize("seed", [0, 1])
def test_oracle_edge_circuit_vs_bigint(seed):
    """CPU pin: the oracle on the edge circuit equals the big-int step model
    (every signal, every cycle, simultaneous commit)."""
    c = edge_circuit(seed)
    n, nl = 4, 3
    staged = _staged(c, n, nl, seed)
    r = oracle.simulate(c, n, n_lanes=nl, staged=staged, watch=list(range(c.n_signals)))
    for l in range(nl):
        regs = {int(x): int(v) for x, v in zip(c.reg_id, c.reg_init)}
        for cyc in range(n):
            vals = R.evaluate(c, {int(s): int(staged[cyc, i, l]) for i, s in enumerate(c.input_id)}, regs)
            assert [int(v) for v in r.trace[cyc, :, l]] == vals, (seed, cyc, l)
            regs = {int(x): vals[int(nx)] % 2 ** int(c.width[int(x)]) for x, nx in zip(c.reg_id, c.reg_next_id)}


def test_edge_circuit_covers_the_corners():
    """The corners the GPU tests rely on are really in the circuit."""
    c = edge_circuit(0)
    op = c.opcode.astype(int)
    ar = np.diff(c.arg_off.astype(np.int64))
    sh = np.isin(op, (9, 10))
    assert {0, 63, 64, 65, 4096} <= set(c.param[sh, 0].tolist())
    a0 = c.arg_id[c.arg_off[:-1]].astype(np.int64)
    assert np.any((op == 3) & (c.width[c.out_id] > c.width[a0]))                  # not widening
    assert np.any((op == 11) & (c.param[:, 0] == 63))                             # bits hi = 63
    a1 = c.arg_id[np.minimum(c.arg_off[:-1] + 1, len(c.arg_id) - 1)].astype(np.int64)
    assert {1, 63, 64} <= set(c.width[a1[op == 12]].tolist())                      # cat w_b
    assert {2, 8, 33, 64} <= set(c.width[a0[op == 13]].tolist())                   # wide selectors
    assert ar.max() == 63 and set(range(4, 9)) - {7} <= set(ar.tolist())           # wide folds


GPU_LANE_CASES = [dict(kernel=1, lane_tile=32), dict(kernel=1, lane_tile=64), dict(kernel=1, lane_tile=128),
                  dict(kernel=1, lane_tile=64, cluster=2), dict(kernel=2, lane_tile=8),
                  dict(kernel=2, lane_tile=16), dict(kernel=2, lane_tile=32, cluster=2),
                  dict(kernel=6, lane_tile=64), dict(kernel=6, lane_tile=128), dict(kernel=6, lane_tile=128, cluster=2),
                  dict(kernel=7, lane_tile=64), dict(kernel=7, lane_tile=128), dict(kernel=7, lane_tile=128, cluster=2),
                  dict(kernel=7, lane_tile=32, op_pairs=2), dict(kernel=7, lane_tile=64, cluster=2, op_pairs=2)]


@pytest.mark.gpu
@pytest.mark.parametrize("kw", GPU_LANE_CASES, ids=lambda k: "-".join(f"{a}{b}" for a, b in k.items()))
@pytest.mark.parametrize("seed", [0, 1])
def test_gpu_edges_lanes(rs, kw, seed):
    c = edge_circuit(seed)
    n, nl = 10, 150
    staged = _staged(c, n, nl, 100 + seed)
    g = rs.Graph(c, device=0)
    L = rs.Lanes(g, nl, lane0=5, stage_cycles=n, **kw)
    assert L.shape()["kernel"] == kw["kernel"]
    L.set_inputs(0, staged)
    H = np.concatenate([L.step(3, hashes="host"), L.step(n - 3, hashes="host")])
    F = L.read(list(range(c.n_signals)))
    r = oracle.simulate(c, n, lane0=5, n_lanes=nl, staged=staged, final=True)
    bad = np.argwhere(H != r.hashes)
    assert bad.shape[0] == 0, f"hash mismatch at (cycle, lane) {bad[:5].tolist()}"
    badf = np.argwhere(F != r.final_state)
    assert badf.shape[0] == 0, f"state mismatch at (signal, lane) {badf[:5].tolist()}"


GPU_SINGLE_CASES = [dict(kernel=3), dict(kernel=3, repcut=2), dict(kernel=4, repcut=2, repcut_global=True),
                    dict(kernel=5), dict(kernel=5, parts=2), dict(kernel=5, parts=3)]


@pytest.mark.gpu
@pytest.mark.parametrize("kw", GPU_SINGLE_CASES, ids=lambda k: "-".join(f"{a}{b}" for a, b in k.items()))
@pytest.mark.parametrize("seed", [0, 1])
def test_gpu_edges_single(rs, kw, seed):
    c = edge_circuit(seed)
    n = 60
    staged = _staged(c, n, 1, 200 + seed)
    kw = dict(kw)
    kernel = kw.pop("kernel")
    g = rs.Graph(c, device=0, mode="single")
    L = rs.Lanes(g, 1, stage_cycles=n, kernel=kernel, **kw)
    assert L.shape()["kernel"] == kernel
    L.set_inputs(0, staged)
    H = np.concatenate([L.step(7, hashes="host"), L.step(n - 7, hashes="host")])
    F = L.read(list(range(c.n_signals)))
    r = oracle.simulate(c, n, n_lanes=1, staged=staged, final=True)
    bad = np.argwhere(H != r.hashes)
    assert bad.shape[0] == 0, f"hash mismatch at (cycle, lane) {bad[:5].tolist()}"
    badf = np.argwhere(F != r.final_state)
    assert badf.shape[0] == 0, f"state mismatch at (signal, lane) {badf[:5].tolist()}"


@pytest.mark.gpu
def test_gpu_edges_seeded_stimulus_all_kernels(rs):
    """Seeded (counter-based) stimulus instead of staged values: uniform values,
    so wide selectors are mostly nonzero -- the complement of the staged mix."""
    c = edge_circuit(2)
    r = oracle.simulate(c, 8, seed=99, lane0=0, n_lanes=70, final=True)
    for kernel in (1, 2, 6, 7):
        g = rs.Graph(c, device=0)
        L = rs.Lanes(g, 70, kernel=kernel)
        L.set_seed(99)
        assert np.array_equal(L.step(8, hashes="host"), r.hashes)
        assert np.array_equal(L.read(list(range(c.n_signals))), r.final_state)
    r1 = oracle.simulate(c, 8, seed=99, n_lanes=1, final=True)
    for kernel in (3, 4, 5):
        g = rs.Graph(c, device=0, mode="single")
        L = rs.Lanes(g, 1, kernel=kernel, **(dict(repcut=1, repcut_global=True) if kernel == 4 else {}))
        L.set_seed(99)
        assert np.array_equal(L.step(8, hashes="host"), r1.hashes), kernel
        assert np.array_equal(L.read(list(range(c.n_signals))), r1.final_state), kernel
