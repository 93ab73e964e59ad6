"""P7 truth tables and P9 invariants of the CPU oracle. CPU only."""
import itertools

import numpy as np
import pytest

import oracle
from synth import GenConfig, config_circuit, fuzz_circuit, generate
from synth.generator import MIX_ALL, CONFIGS
from tests import bigint_ref as R


def tiny_comb(seed: int, in_widths, n_ops=24, n_levels=4):
    cfg = GenConfig(f"tiny{seed}", n_ops, n_levels, 0, len(in_widths), tuple(MIX_ALL), "u1_16",
                    0.2, 500 + seed, 0, 1, 1, n_consts=1)
    c = generate(cfg)
    w = c.width.copy()
    w[c.input_id] = np.array(in_widths, dtype=np.uint8)
    c.width = w
    return c.normalized()


@pytest.mark.parametrize("seed,in_widths", [(0, (3, 3, 3)), (1, (4, 5)), (2, (1, 2, 3, 3)),
                                             (3, (6, 6)), (4, (2, 2, 2, 2, 1))])
def test_truth_table_vs_bigint(seed, in_widths):
    """P7: every input combination of a tiny random combinational circuit
    (all 2^k as lanes) vs the big-integer evaluator, on every signal."""
    c = tiny_comb(seed, in_widths)
    combos = list(itertools.product(*[range(2 ** w) for w in in_widths]))
    L = len(combos)
    staged = np.array(combos, dtype=np.uint64).T[None]             # [1][n_inputs][L]
    r = oracle.simulate(c, 1, n_lanes=L, staged=staged, final=True, hashes=False)
    for l, combo in enumerate(combos):
        ref = R.evaluate(c, {int(s): v for s, v in zip(c.input_id, combo)})
        got = [int(v) for v in r.final_state[:, l]]
        assert got == ref, (seed, combo)


def test_truth_table_16_input_bits():
    """P7 at 16 input bits (65,536 lanes), checked on a sample of lanes plus a
    full-table check of the hash against the big-int evaluator's hash."""
    c = tiny_comb(9, (8, 8), n_ops=16, n_levels=3)
    A = np.repeat(np.arange(256, dtype=np.uint64), 256)
    B = np.tile(np.arange(256, dtype=np.uint64), 256)
    r = oracle.simulate(c, 1, n_lanes=65536, staged=np.stack([A, B])[None], final=True)
    rng = np.random.default_rng(0)
    K = [oracle.hash_weight(s) for s in range(c.n_signals)]
    for l in rng.choice(65536, size=300, replace=False):
        ref = R.evaluate(c, {int(c.input_id[0]): int(A[l]), int(c.input_id[1]): int(B[l])})
        assert [int(v) for v in r.final_state[:, l]] == ref
        assert int(r.hashes[0, l]) == sum(v * k for v, k in zip(ref, K)) % 2 ** 64


@pytest.mark.parametrize("seed", range(0, 40))
def test_fuzz_corpus_vs_bigint_multicycle(seed):
    """Fuzz corpus members (constants, register->source edges, wide folds,
    permuted ids): 6 cycles of the oracle vs a big-int step-by-step model
    with simultaneous commit."""
    c = fuzz_circuit(seed)
    n = 6
    rng = np.random.default_rng(seed)
    staged = rng.integers(0, 2**63, size=(n, c.n_inputs, 2), dtype=np.int64).astype(np.uint64)
    r = oracle.simulate(c, n, n_lanes=2, staged=staged, watch=list(range(c.n_signals)))
    for l in range(2):
        regs = {int(x): int(v) for x, v in zip(c.reg_id, c.reg_init)}
        for cyc in range(n):
            vals = R.evaluate(c, {int(s): int(staged[cyc, i, l]) for i, s in enumerate(c.input_id)},
                              regs)
            assert [int(v) for v in r.trace[cyc, :, l]] == vals, (seed, cyc)
            regs = {int(x): vals[int(nx)] % 2 ** int(c.width[int(x)])
                    for x, nx in zip(c.reg_id, c.reg_next_id)}


def _scaled(name, **kw):
    return config_circuit(name, **kw)


def test_mask_invariant_and_activity():
    """P9 mask invariant v <= M(w); SURVEY.md §8(d) activity check: fewer than
    50% of signals constant over cycles 50..100 (else parity is vacuous)."""
    for name, kw in (("C2", {}), ("C3", dict(n_ops=15000, n_levels=80, n_regs=2000))):
        c = _scaled(name, **kw)
        r = oracle.simulate(c, 101, seed=CONFIGS[name].stim_seed, n_lanes=4,
                            watch=list(range(c.n_signals)), threads=4, hashes=False)
        T = r.trace
        w = c.width.astype(np.uint64)
        lim = np.where(w >= 64, np.uint64(2**64 - 1), (np.uint64(1) << np.minimum(w, 63)) - np.uint64(1))
        assert (T <= lim[None, :, None]).all()
        const = (T[50:] == T[50][None]).all(axis=(0, 2))
        assert const.mean() < 0.5, (name, const.mean())


def test_operand_order_sensitivity():
    """P9 / SPEC.md S:346: reversing the O order of sub/cat changes results."""
    c = _scaled("C2", n_ops=3000, n_levels=12, n_regs=200)
    h0 = oracle.simulate(c, 20, seed=5, n_lanes=2).hashes
    c2 = c.normalized()
    for j in np.nonzero((c2.opcode == R.SUB) | (c2.opcode == R.CAT))[0]:
        a, b = c2.arg_off[j], c2.arg_off[j + 1]
        c2.arg_id[a:b] = c2.arg_id[a:b][::-1]
    h1 = oracle.simulate(c2, 20, seed=5, n_lanes=2).hashes
    assert not np.array_equal(h0, h1)


def test_op_list_order_and_id_permutation_invariance():
    """P9: the op list order is irrelevant (the oracle finds its own
    topological order); renaming signals permutes values (hash weights are
    per canonical id, so hashes change with ids but values do not)."""
    c = _scaled("C2", n_ops=2000, n_levels=10, n_regs=100)
    r0 = oracle.simulate(c, 15, seed=9, n_lanes=3, final=True)
    p = np.random.default_rng(1).permutation(c.n_ops)
    arity = np.diff(c.arg_off.astype(np.int64))
    args = [c.arg_id[c.arg_off[j]:c.arg_off[j + 1]] for j in p]
    c1 = c.normalized()
    c1.opcode, c1.out_id, c1.param = c.opcode[p], c.out_id[p], c.param[p]
    c1.arg_off = np.concatenate([[0], np.cumsum(arity[p])]).astype(np.uint32)
    c1.arg_id = np.concatenate(args).astype(np.uint32)
    c1.level = None
    r1 = oracle.simulate(c1.normalized(), 15, seed=9, n_lanes=3, final=True)
    assert np.array_equal(r0.hashes, r1.hashes)
    perm = np.random.default_rng(2).permutation(c.n_signals)
    cp = c.permuted(perm)
    rp = oracle.simulate(cp, 15, seed=9, n_lanes=3, final=True)
    assert np.array_equal(rp.final_state[perm], r0.final_state)


def test_lane_independence_and_chunking():
    """P9: a lane run alone equals the same lane in a batch; splitting the run
    (resume from committed registers at cycle0) equals one run."""
    c = _scaled("C2", n_ops=3000, n_levels=15, n_regs=300)
    full = oracle.simulate(c, 40, seed=3, lane0=100, n_lanes=8, final=True)
    alone = oracle.simulate(c, 40, seed=3, lane0=105, n_lanes=1)
    assert np.array_equal(full.hashes[:, 5], alone.hashes[:, 0])
    a = oracle.simulate(c, 25, seed=3, lane0=100, n_lanes=8, final=True)
    regs0 = a.final_state[c.reg_id]
    b = oracle.simulate(c, 15, seed=3, lane0=100, n_lanes=8, cycle0=25, reg_state0=regs0, final=True)
    assert np.array_equal(np.concatenate([a.hashes, b.hashes]), full.hashes)
    assert np.array_equal(b.final_state, full.final_state)
    sampled = oracle.simulate(c, 40, seed=3, lanes=[100, 103, 104, 107])
    assert np.array_equal(sampled.hashes, full.hashes[:, [0, 3, 4, 7]])


def test_topo_errors():
    from synth import Builder
    b = Builder()
    x = b.input(4)
    y = b.op("add", [x, x], 4)
    c = b.build()
    c.arg_id[0] = y                          # self loop
    with pytest.raises(ValueError):
        oracle.topo_order(c)
    c = b.build()
    c.out_id[0] = x                          # two drivers
    with pytest.raises(ValueError):
        oracle.topo_order(c)
