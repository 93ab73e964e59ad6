"""Hand-built circuits whose behaviour has a closed form (SURVEY.md §8(c)
pins P1-P6).  Structure only: the expected values live in the tests.
"""
from __future__ import annotations

from typing import List, Tuple

from .circuit import Builder, Circuit


def paper_example(two_muls: bool = False) -> Tuple[Circuit, List[int]]:
    """PAPER.md Fig. DFG-a / fig:Rrank: register inputs 1, 2, 4
    form LI (rank R); OIM selects 1 and 4, reduced by multiply -> 4.  With
    ``two_muls`` an S rank of shape 2 is added (Fig. DFG-b);
    the second multiply's operands (2, 4) are our choice (the figure is absent).
    Registers hold their value (next = self)."""
    b = Builder("paper_fig6")
    r = [b.reg(8, v) for v in (1, 2, 4)]
    for x in r:
        b.set_next(x, x)
    outs = [b.op("mul", [r[0], r[2]], 8)]
    if two_muls:
        outs.append(b.op("mul", [r[1], r[2]], 8))
    return b.build(), outs


def counter(w: int) -> Tuple[Circuit, int]:
    """r <- add(r, 1) at width w."""
    b = Builder(f"counter{w}")
    r = b.reg(w, 0)
    one = b.const(w, 1)
    b.set_next(r, b.op("add", [r, one], w))
    return b.build(), r


def accumulator(w: int, w_in: int) -> Tuple[Circuit, int, int]:
    """r <- add(r, in): the iterative-rank prefix sum S_{i+1} = S_i + A_i
    (PAPER.md eq:iter:s P:403-405, alg:prefix-sum P:408-415)."""
    b = Builder(f"acc{w}")
    x = b.input(w_in)
    r = b.reg(w, 0)
    b.set_next(r, b.op("add", [r, x], w))
    return b.build(), r, x


def ripple_adder(n: int) -> Tuple[Circuit, int, int, int]:
    """n-bit ripple-carry adder from bits / 1-bit xor, and, or / cat:
    out = a + b as an (n+1)-bit value.  Depth ~2n levels."""
    b = Builder(f"ripple{n}")
    a = b.input(n)
    c = b.input(n)
    carry = None
    sums = []
    for i in range(n):
        ai = b.op("bits", [a], 1, i, i)
        ci = b.op("bits", [c], 1, i, i)
        if carry is None:
            s = b.op("xor", [ai, ci], 1)
            carry = b.op("and", [ai, ci], 1)
        else:
            t = b.op("xor", [ai, ci], 1)
            s = b.op("xor", [t, carry], 1)
            g = b.op("and", [ai, ci], 1)
            p = b.op("and", [t, carry], 1)
            carry = b.op("or", [g, p], 1)
        sums.append(s)
    acc = carry                                 # MSB first: cat(high, low)
    w = 1
    for s in reversed(sums):
        w += 1
        acc = b.op("cat", [acc, s], w)
    return b.build(), a, c, acc


def lfsr(nbits: int, taps: Tuple[int, ...], seed: int = 1) -> Tuple[Circuit, int]:
    """Fibonacci LFSR, shift left, feedback = xor of the tap bits (taps are
    1-based bit positions, e.g. (16, 14, 13, 11)); maximal taps give period
    2^n - 1."""
    b = Builder(f"lfsr{nbits}")
    s = b.reg(nbits, seed)
    tb = [b.op("bits", [s], 1, t - 1, t - 1) for t in taps]
    fb = tb[0] if len(tb) == 1 else b.op("xor", tb, 1)
    low = b.op("bits", [s], nbits - 1, nbits - 2, 0)
    b.set_next(s, b.op("cat", [low, fb], nbits))
    return b.build(), s


def shift_register(depth: int, w: int) -> Tuple[Circuit, int, List[int]]:
    """r0 <- in, r_k <- r_{k-1}: needs the simultaneous commit."""
    b = Builder(f"shreg{depth}")
    x = b.input(w)
    rs = [b.reg(w, 0) for _ in range(depth)]
    b.set_next(rs[0], x)
    for k in range(1, depth):
        b.set_next(rs[k], rs[k - 1])
    return b.build(), x, rs


def swap(w: int, a0: int, b0: int) -> Tuple[Circuit, int, int]:
    """r1 <- r2, r2 <- r1."""
    b = Builder("swap")
    r1 = b.reg(w, a0)
    r2 = b.reg(w, b0)
    b.set_next(r1, r2)
    b.set_next(r2, r1)
    return b.build(), r1, r2
