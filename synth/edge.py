"""Edge-case circuits and staged edge values for GPU parity (structure only).

Every op of the method's vocabulary at the corners of its semantics
(readings R1-R5), wired so the corner values propagate through
several levels and across cycles through registers:

* shl / shr with amounts n in {0, 1, w-1, w, 63, 64, 65, 4096} (n >= 64 gives
  0, reading R5) and out widths narrower / wider than the operand;
* not into an out width wider than its operand (reading R3: the upper bits
  become 1) and narrower;
* bits with hi = 63 and lo in {0, 31, 63}, and hi = lo;
* cat with w_b = w(x1) in {1, 63, 64} (w_b = 64 returns x1, reading R5);
* mux with multi-bit selectors (2, 8, 33, 64 bits; nonzero picks O=1,
  reading R4), including selectors that are often zero;
* and/or/xor/add/sub/mul folds of 4..8 operands and one of 63 operands (the
  ABI maximum) over mixed widths (left fold in O order, PAPER.md
  eq:custom_reduce P:778-796);
* eq / lt over operands of different widths, declared out widths > 1.

``edge_values`` draws staged input values biased to 0, all ones, 1, 2^63 and
sparse bit patterns, so selectors are often zero and shifts / compares hit
their boundaries.  Nothing here evaluates an op.
"""
from __future__ import annotations

import numpy as np

from .circuit import Builder, Circuit

IN_WIDTHS = (1, 2, 7, 8, 9, 15, 16, 17, 31, 32, 33, 63, 64)
SHIFTS = (0, 1, "w-1", "w", 63, 64, 65, 4096)


def edge_circuit(seed: int = 0, layers: int = 3) -> Circuit:
    rng = np.random.default_rng(7000 + seed)
    b = Builder(f"edge{seed}")
    pool = [b.input(w) for w in IN_WIDTHS]
    regs = [b.reg(w, init=int(rng.integers(0, 2**63))) for w in (1, 8, 33, 64, 17, 2)]
    pool += regs
    W = b.width

    def pick(k=1, widths=None):
        cand = [s for s in pool if widths is None or W[s] in widths]
        return [int(x) for x in rng.choice(cand, size=k, replace=len(cand) < k)]

    for layer in range(layers):
        new = []
        # shifts at every boundary, out narrower / equal / wider
        for x in pick(6):
            w = W[x]
            for n in SHIFTS:
                nn = w - 1 if n == "w-1" else w if n == "w" else n
                for wo in {1, w, 64, int(rng.integers(1, 65))}:
                    new.append(b.op("shl", [x], wo, p0=nn))
                    new.append(b.op("shr", [x], wo, p0=nn))
        # not widening / narrowing
        for x in pick(5, widths=(1, 2, 7, 9, 31, 33, 63)):
            w = W[x]
            for wo in {w, min(64, w + 1), 64, 1}:
                new.append(b.op("not", [x], wo))
        # bits with hi = 63, hi = lo
        for x in pick(4, widths=(63, 64)):
            for hi, lo in ((63, 0), (63, 31), (63, 63), (40, 40), (0, 0)):
                for wo in {hi - lo + 1, 64, 1}:
                    new.append(b.op("bits", [x], wo, p0=hi, p1=lo))
        # cat with w_b in {1, 63, 64}
        for wb in (1, 63, 64):
            for x0 in pick(3):
                x1 = pick(1, widths=(wb,))[0]
                for wo in {64, min(64, W[x0] + wb), 8}:
                    new.append(b.op("cat", [x0, x1], wo))
        # mux with multi-bit selectors
        for ws in (2, 8, 33, 64):
            for _ in range(3):
                sel = pick(1, widths=(ws,))[0]
                a, c = pick(2)
                for wo in (1, 16, 64):
                    new.append(b.op("mux", [sel, a, c], wo))
        # wide folds (O rank > 3) and one of the ABI maximum 63
        for opn in ("and", "or", "xor", "add", "sub", "mul"):
            for ar in (4, 5, 6, 8):
                new.append(b.op(opn, pick(ar), int(rng.choice([1, 17, 64, int(rng.integers(1, 65))]))))
            if layer == 0:
                new.append(b.op(opn, pick(63), 64))
        # mixed-width compares with declared widths > 1; 2-operand arithmetic into 1 bit
        for opn in ("eq", "lt"):
            for _ in range(6):
                new.append(b.op(opn, pick(2), int(rng.choice([1, 5, 64]))))
        for opn in ("add", "sub", "mul", "and", "or", "xor"):
            for _ in range(3):
                new.append(b.op(opn, pick(2), int(rng.choice([1, 64]))))
        pool += new
    # registers take corner values across cycles
    ops_out = [s for s in pool if s not in regs and s >= len(IN_WIDTHS) + len(regs)]
    for r in regs:
        b.set_next(r, int(rng.choice(ops_out)))
    return b.build()


def edge_values(rng: np.random.Generator, shape) -> np.ndarray:
    """Staged input values (u64) biased to the corners; the library and the
    oracle both mask them to each input's width."""
    n = int(np.prod(shape))
    kind = rng.integers(0, 100, size=n)
    rand = rng.integers(0, 2**63, size=n, dtype=np.int64).astype(np.uint64) * np.uint64(2) \
        + rng.integers(0, 2, size=n).astype(np.uint64)
    sparse = np.uint64(1) << rng.integers(0, 64, size=n).astype(np.uint64)
    v = np.where(kind < 25, np.uint64(0),
        np.where(kind < 40, np.uint64(0xFFFFFFFFFFFFFFFF),
        np.where(kind < 50, np.uint64(1),
        np.where(kind < 55, np.uint64(1) << np.uint64(63),
        np.where(kind < 70, sparse, rand)))))
    return v.reshape(shape)


def pass_circuit(seed: int = 0, n: int = 400) -> Circuit:
    """A random circuit rich in what the compiler's graph passes remove (SURVEY.md
    §8(f) NEXT-1): constants feeding ops (constant propagation), identity ops --
    shifts by 0, full-width bits, and with all ones, or / xor / add with 0, sub of
    0, mul by 1, mux with a constant selector or equal branches, cat(0, x) -- and
    absorbing ones (and with 0, x ^ x, x - x, eq(x, x)), in chains, feeding
    registers and each other, mixed with ordinary ops.  Structure only."""
    rng = np.random.default_rng(9000 + seed)
    b = Builder(f"passes{seed}")
    pool = [b.input(int(w)) for w in rng.choice([1, 4, 8, 13, 32, 64], size=6)]
    regs = [b.reg(int(w), init=int(rng.integers(0, 2**40))) for w in (1, 8, 32, 64, 5)]
    pool += regs
    consts = [b.const(w, v) for w, v in ((64, 0), (64, 2**64 - 1), (8, 1), (1, 1), (1, 0), (16, 0xABCD), (64, 1))]
    W = b.width
    zero64, ones64, one8, one1, zero1, k16, one64 = consts

    def pick():
        return int(rng.choice(pool))

    for _ in range(n):
        x = pick()
        w = W[x]
        kind = int(rng.integers(0, 18))
        if kind == 0:
            s = b.op("shl", [x], w + int(rng.integers(0, 65 - w)), p0=0)
        elif kind == 1:
            s = b.op("shr", [x], w, p0=0)
        elif kind == 2:
            s = b.op("bits", [x], w, p0=min(63, w - 1 + int(rng.integers(0, 3))), p1=0)
        elif kind == 3:
            s = b.op("and", [x, ones64] if rng.random() < 0.5 else [ones64, x], w)
        elif kind == 4:
            s = b.op(str(rng.choice(["or", "xor", "add"])), [x, zero64] if rng.random() < 0.5 else [zero64, x], 64)
        elif kind == 5:
            s = b.op("sub", [x, zero64], w)
        elif kind == 6:
            s = b.op("mul", [x, one64], w)
        elif kind == 7:
            s = b.op("mux", [int(rng.choice([one1, zero1, k16, zero64])), x, pick()], 64)
        elif kind == 8:
            s = b.op("mux", [pick(), x, x], w)
        elif kind == 9:
            s = b.op("cat", [zero64, x], w)
        elif kind == 10:
            s = b.op(str(rng.choice(["and", "mul"])), [x, zero64], w)
        elif kind == 11:
            s = b.op(str(rng.choice(["xor", "sub", "eq", "lt", "or", "and"])), [x, x], w)
        elif kind == 12:
            s = b.op(str(rng.choice(["add", "xor", "mul", "eq", "lt", "cat"])),
                     [int(rng.choice(consts)), int(rng.choice(consts))], int(rng.integers(1, 65)))
        elif kind == 13:
            s = b.op("not", [int(rng.choice(consts))], int(rng.integers(1, 65)))
        else:
            s = b.op(str(rng.choice(["add", "xor", "and", "or", "sub", "mul", "eq", "lt", "cat"])), [x, pick()],
                     int(rng.integers(1, 65)))
        pool.append(s)
    ops_out = [s for s in pool[len(pool) - n:]]
    for r in regs:
        b.set_next(r, int(rng.choice(ops_out)))
    return b.build()
