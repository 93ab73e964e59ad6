"""Independent definitions of the op semantics in Python arbitrary-precision
integers -- used only to pin the C oracle (SURVEY.md §8(c) pins P7/P8).

These are written as the FIRRTL *mathematical* definitions (integer
arithmetic followed by reduction modulo 2**w), using //, % and * by powers of
two instead of the oracle's shifts and masks, so a wrong shift edge case, a
missing mask or a transposed operand in the C code fails against them.
"""
from __future__ import annotations

from typing import Dict, List, Sequence

AND, OR, XOR, NOT, ADD, SUB, MUL, EQ, LT, SHL, SHR, BITS, CAT, MUX = range(14)


def mod(x: int, w: int) -> int:
    return x % (2 ** w)


def op_ref(opc: int, xs: Sequence[int], w_out: int, p0: int = 0, p1: int = 0, wb: int = 0) -> int:
    xs = [int(x) for x in xs]
    if opc in (AND, OR, XOR):
        r = xs[0]
        for x in xs[1:]:
            r = (r & x) if opc == AND else (r | x) if opc == OR else (r ^ x)
        return mod(r, w_out)
    if opc == ADD:
        return mod(sum(xs), w_out)
    if opc == SUB:                      # left fold in O order
        r = xs[0]
        for x in xs[1:]:
            r = r - x
        return mod(r, w_out)
    if opc == MUL:
        r = 1
        for x in xs:
            r = r * x
        return mod(r, w_out)
    if opc == EQ:
        return mod(1 if xs[0] == xs[1] else 0, w_out)
    if opc == LT:
        return mod(1 if xs[0] < xs[1] else 0, w_out)
    if opc == NOT:                      # complement within the 64-bit value domain
        return mod((2 ** 64 - 1) - xs[0], w_out)
    if opc == SHL:                      # FIRRTL x * 2^n, truncated to w_out (<= 64)
        return mod(xs[0] * (2 ** p0), w_out)
    if opc == SHR:
        return mod(xs[0] // (2 ** p0), w_out)
    if opc == BITS:
        return mod(mod(xs[0] // (2 ** p1), p0 - p1 + 1), w_out)
    if opc == CAT:
        return mod(xs[0] * (2 ** wb) + xs[1], w_out)   # x0 is the high part
    if opc == MUX:
        return mod(xs[1] if xs[0] != 0 else xs[2], w_out)
    raise ValueError(opc)


def evaluate(circ, input_values: Dict[int, int], reg_values: Dict[int, int] = None) -> List[int]:
    """Evaluate one combinational pass of ``circ`` (any op order that respects
    dependencies; found here by repeated sweeps) and return all signal values."""
    n = circ.n_signals
    val: List = [None] * n
    for s, v in input_values.items():
        val[s] = mod(v, int(circ.width[s]))
    for i, r in enumerate(circ.reg_id):
        r = int(r)
        v = reg_values[r] if reg_values and r in reg_values else int(circ.reg_init[i])
        val[r] = mod(v, int(circ.width[r]))
    for i, s in enumerate(circ.const_id):
        val[int(s)] = mod(int(circ.const_val[i]), int(circ.width[int(s)]))
    pending = list(range(circ.n_ops))
    while pending:
        rest = []
        for j in pending:
            args = circ.op_args(j)
            if any(val[a] is None for a in args):
                rest.append(j)
                continue
            wb = int(circ.width[args[1]]) if len(args) >= 2 else 0
            val[int(circ.out_id[j])] = op_ref(int(circ.opcode[j]), [val[a] for a in args],
                                              int(circ.width[int(circ.out_id[j])]),
                                              int(circ.param[j, 0]), int(circ.param[j, 1]), wb)
        if len(rest) == len(pending):
            raise ValueError("combinational loop")
        pending = rest
    return val
