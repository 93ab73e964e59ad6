"""Pins of the CPU oracle against what the paper and mathematics fix
(SURVEY.md §8(c) P1-P9).  CPU only."""
import itertools

import numpy as np
import pytest

import oracle
from synth import Builder, closed_form as cf
from synth.circuit import OP_NAMES
from tests import bigint_ref as R

pytestmark = pytest.mark.filterwarnings("ignore")
M64 = 2 ** 64 - 1


# ---------------------------------------------------------------- stimulus / hash
def test_splitmix64_published_vector():
    """splitmix64 reference outputs for seed 1234567 (public test vector of the
    algorithm, Steele/Lea/Flood 2014; Vigna's splitmix64.c): the generator's
    n-th output is next(seed + (n-1)*gamma)."""
    expect = [6457827717110365317, 3203168211198807973, 9817491932198370423,
              4593380528125082431, 16408922859458223821]
    gamma = 0x9E3779B97F4A7C15
    got = [oracle.splitmix_next((1234567 + n * gamma) & M64) for n in range(5)]
    assert got == expect


def test_stimulus_composition_and_golden():
    """Reading R13: stim = next(next(next(next(seed)+k)+c)+lane); the golden
    file was written by tests/golden/make_golden.py (oracle only)."""
    import json, os
    nx = oracle.splitmix_next
    for (s, k, c, l) in [(0, 0, 0, 0), (202, 5, 77, 1000), (M64, 3, 2**40, 7)]:
        assert oracle.stimulus(s, k, c, l) == nx((nx((nx((nx(s) + k) & M64) + c) & M64) + l) & M64)
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "stimulus_seed1.json")))
    for row in g["values"]:
        assert oracle.stimulus(g["seed"], row["k"], row["c"], row["lane"]) == int(row["value"])


def test_hash_weights_odd_and_distinct():
    K = [oracle.hash_weight(s) for s in range(5000)]
    assert all(k & 1 for k in K)
    assert len(set(K)) == len(K)


# ---------------------------------------------------------------- P1 paper example
def test_paper_worked_example_single_multiply():
    """P1: PAPER.md Fig. DFG-a / fig:Rrank caption: LI = [1, 2, 4];
    OIM selects 1 and 4; the product stored in LO is 4."""
    c, outs = cf.paper_example()
    r = oracle.simulate(c, 1, watch=outs)
    assert int(r.trace[0, 0, 0]) == 4


def test_paper_worked_example_two_multiplies():
    """Fig. DFG-b / fig:Srank: S rank of shape 2 -> two outputs."""
    c, outs = cf.paper_example(two_muls=True)
    r = oracle.simulate(c, 3, watch=outs)
    assert r.trace.shape[1] == 2
    assert [int(v) for v in r.trace[0, :, 0]] == [4, 8]
    assert (r.trace == r.trace[0]).all()          # registers hold: same every cycle


# ---------------------------------------------------------------- P8 per-op semantics
def _apply(opc, xs, w, p0=0, p1=0, wb=0):
    return oracle.apply_op(opc, xs, w, p0, p1, wb)


@pytest.mark.parametrize("opc", range(14))
def test_ops_exhaustive_small_widths(opc):
    """P8: every operand pair at 3-bit widths and every out width 1..6 (and
    shift/bits/cat parameter sweeps) vs the big-integer definition."""
    vals = range(8)
    for w in range(1, 7):
        if opc in (R.NOT, R.SHL, R.SHR, R.BITS):
            for x in vals:
                if opc == R.BITS:
                    for lo in range(0, 3):
                        for hi in range(lo, 4):
                            assert _apply(opc, [x], w, hi, lo) == R.op_ref(opc, [x], w, hi, lo)
                elif opc in (R.SHL, R.SHR):
                    for n in (0, 1, 2, 3, 5, 63, 64, 65, 1000):
                        assert _apply(opc, [x], w, n) == R.op_ref(opc, [x], w, n)
                else:
                    assert _apply(opc, [x], w) == R.op_ref(opc, [x], w)
        elif opc == R.MUX:
            for s, a, b in itertools.product(range(4), vals, vals):
                assert _apply(opc, [s, a, b], w) == R.op_ref(opc, [s, a, b], w)
        else:
            for a, b in itertools.product(vals, vals):
                wb = 3
                assert _apply(opc, [a, b], w, 0, 0, wb) == R.op_ref(opc, [a, b], w, 0, 0, wb), \
                    (OP_NAMES[opc], a, b, w)


def test_ops_exhaustive_8bit_vectorized():
    """P8 at 8-bit operands: all 65,536 pairs, every out width 1..8, through a
    one-cycle circuit (staged inputs as lanes) vs exact int64 definitions."""
    b = Builder("ops8")
    x = b.input(8)
    y = b.input(8)
    outs = []
    for w in range(1, 9):
        for name in ("and", "or", "xor", "add", "sub", "mul", "eq", "lt", "cat"):
            outs.append((name, w, b.op(name, [x, y], w if name not in ("eq", "lt") else 1)))
        outs.append(("not", w, b.op("not", [x], w)))
        outs.append(("mux", w, b.op("mux", [x, x, y], w)))
    c = b.build()
    a = np.repeat(np.arange(256, dtype=np.int64), 256)
    d = np.tile(np.arange(256, dtype=np.int64), 256)
    staged = np.stack([a, d])[None].astype(np.uint64)
    r = oracle.simulate(c, 1, n_lanes=65536, staged=staged, watch=[o[2] for o in outs],
                        hashes=False)
    for i, (name, w, _) in enumerate(outs):
        m = 2 ** w
        ref = {"and": a & d, "or": a | d, "xor": a ^ d, "add": (a + d) % m, "sub": (a - d) % m,
               "mul": (a * d) % m, "eq": (a == d).astype(np.int64), "lt": (a < d).astype(np.int64),
               "cat": (a * 256 + d) % m, "not": (255 - a) % m if w <= 8 else None,
               "mux": np.where(a != 0, a, d) % m}[name]
        if name in ("and", "or", "xor"):
            ref = ref % m
        assert np.array_equal(r.trace[0, i].astype(np.int64), ref), (name, w)


EDGE = [0, 1, 2, 3, 2**31 - 1, 2**31, 2**32 - 1, 2**32, 2**63 - 1, 2**63, 2**64 - 2, M64,
        0x0123456789ABCDEF, 0xFEDCBA9876543210]


@pytest.mark.parametrize("opc", range(14))
def test_ops_edges_64bit(opc):
    """P8 edges at 64 bits: M(64), shifts 63/64/65, cat with w_b = 64, bits hi = 63,
    sub wrap, mul overflow, 3-operand folds (O order)."""
    rng = np.random.default_rng(opc)
    for w in (1, 7, 31, 32, 33, 63, 64):
        for a in EDGE:
            for b in EDGE[::3]:
                if opc in (R.NOT,):
                    xs, ps = [a], [(0, 0, 0)]
                elif opc in (R.SHL, R.SHR):
                    xs, ps = [a], [(n, 0, 0) for n in (0, 1, 31, 32, 63, 64, 65, 4096)]
                elif opc == R.BITS:
                    xs, ps = [a], [(63, 0, 0), (63, 63, 0), (40, 8, 0), (31, 0, 0), (0, 0, 0), (63, 32, 0)]
                elif opc == R.CAT:
                    ps = [(0, 0, wb) for wb in (1, 8, 32, 63, 64)]
                    xs = None
                elif opc == R.MUX:
                    xs, ps = [a & 1, a, b], [(0, 0, 0)]
                else:
                    xs, ps = [a, b], [(0, 0, 0)]
                for (p0, p1, wb) in ps:
                    xx = xs if xs is not None else [a, b % (2 ** wb)]
                    assert _apply(opc, xx, w, p0, p1, wb) == R.op_ref(opc, xx, w, p0, p1, wb), \
                        (OP_NAMES[opc], xx, w, p0, p1, wb)
    if opc in (R.AND, R.OR, R.XOR, R.ADD, R.SUB, R.MUL):
        for _ in range(200):
            xs = [int(v) for v in rng.integers(0, 2**63, size=int(rng.integers(2, 6)), dtype=np.int64)]
            xs = [x * 2 + 1 if x % 3 == 0 else x for x in xs]
            w = int(rng.integers(1, 65))
            assert _apply(opc, xs, w) == R.op_ref(opc, xs, w)


def test_sub_operand_order_and_spec_example():
    """O-order sensitivity: sub(2,5) at 4 bits = 13,
    sub(5,2) = 3; 3-operand sub is a left fold ((x0-x1)-x2)."""
    assert _apply(R.SUB, [2, 5], 4) == 13
    assert _apply(R.SUB, [5, 2], 4) == 3
    assert _apply(R.SUB, [10, 3, 2], 8) == 5
    assert _apply(R.MUX, [1, 7, 2], 4) == 7
    assert _apply(R.MUX, [0, 7, 2], 4) == 2
    assert _apply(R.MUL, [1, 4], 4) == 4              # SPEC.md S:300 / PAPER P:681


# ---------------------------------------------------------------- P2-P6 closed forms
@pytest.mark.parametrize("w", [1, 3, 8, 13, 64])
def test_counter(w):
    """P2: r <- r + 1 at width w: pre-commit value at cycle c is c mod 2^w."""
    c, r = cf.counter(w)
    n = 300
    t = oracle.simulate(c, n, watch=[r]).trace[:, 0, 0]
    assert [int(v) for v in t] == [k % (2 ** w) for k in range(n)]


@pytest.mark.parametrize("w,w_in", [(8, 8), (16, 5), (64, 64), (3, 7)])
def test_accumulator_is_prefix_sum(w, w_in):
    """P3: r <- r + in is the paper's iterative-rank prefix sum (eq:iter:s,
    alg:prefix-sum P:401-415): r_c = sum_{j<c} in_j mod 2^w, with staged
    random inputs on 5 lanes."""
    c, r, x = cf.accumulator(w, w_in)
    rng = np.random.default_rng(7)
    n, L = 200, 5
    vals = rng.integers(0, 2**63, size=(n, 1, L), dtype=np.int64).astype(np.uint64) * np.uint64(2)
    t = oracle.simulate(c, n, n_lanes=L, staged=vals, watch=[r]).trace[:, 0, :]
    ins = [[int(vals[j, 0, l]) % (2 ** w_in) for j in range(n)] for l in range(L)]
    for l in range(L):
        for k in range(n):
            assert int(t[k, l]) == sum(ins[l][:k]) % (2 ** w)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_ripple_adder_exhaustive(n):
    """P4: an n-bit ripple-carry adder of bits/xor/and/or/cat equals integer
    a + b, for all (a, b) (65,536 lanes at n = 8)."""
    c, a, b, out = cf.ripple_adder(n)
    A = np.repeat(np.arange(2**n, dtype=np.uint64), 2**n)
    B = np.tile(np.arange(2**n, dtype=np.uint64), 2**n)
    r = oracle.simulate(c, 1, n_lanes=A.size, staged=np.stack([A, B])[None], watch=[out], hashes=False)
    assert np.array_equal(r.trace[0, 0], A + B)


@pytest.mark.parametrize("n", [32, 63])
def test_ripple_adder_random_wide(n):
    c, a, b, out = cf.ripple_adder(n)
    rng = np.random.default_rng(n)
    L = 512
    A = rng.integers(0, 2**62, size=L, dtype=np.int64).astype(np.uint64) * np.uint64(2) % np.uint64(2**n)
    B = rng.integers(0, 2**62, size=L, dtype=np.int64).astype(np.uint64) * np.uint64(3) % np.uint64(2**n)
    r = oracle.simulate(c, 1, n_lanes=L, staged=np.stack([A, B])[None], watch=[out], hashes=False)
    got = [int(v) for v in r.trace[0, 0]]
    assert got == [int(x) + int(y) for x, y in zip(A, B)]


@pytest.mark.parametrize("nbits,taps", [(4, (4, 3)), (8, (8, 6, 5, 4)), (16, (16, 14, 13, 11))])
def test_lfsr_maximal_period(nbits, taps):
    """P5: maximal-length Fibonacci LFSR taps give period exactly 2^n - 1 and
    visit every nonzero state once."""
    c, s = cf.lfsr(nbits, taps, seed=1)
    P = 2 ** nbits - 1
    t = [int(v) for v in oracle.simulate(c, P + 1, watch=[s], hashes=False).trace[:, 0, 0]]
    assert t[0] == 1 and t[P] == 1
    assert len(set(t[:P])) == P and 0 not in t


def test_shift_register_simultaneous_commit():
    """P6: r0 <- in, r_k <- r_{k-1}: r_k(c) = in(c-1-k), 0 before the fill."""
    depth = 6
    c, x, rs = cf.shift_register(depth, 16)
    n = 40
    vals = (np.arange(n, dtype=np.uint64) * np.uint64(977) + np.uint64(5))[:, None, None]
    t = oracle.simulate(c, n, staged=vals, watch=rs).trace[:, :, 0]
    for cyc in range(n):
        for k in range(depth):
            j = cyc - 1 - k
            assert int(t[cyc, k]) == (int(vals[j, 0, 0]) % 2**16 if j >= 0 else 0)


def test_swap_exchanges_each_cycle():
    """P6: r1 <- r2, r2 <- r1 exchange every cycle."""
    c, r1, r2 = cf.swap(8, 3, 200)
    t = oracle.simulate(c, 5, watch=[r1, r2]).trace[:, :, 0]
    assert [tuple(int(v) for v in row) for row in t] == [(3, 200), (200, 3)] * 2 + [(3, 200)]
