"""Circuit description shared by the oracle side and the CUDA side.

This module holds only the *interchange format* of a synchronous circuit
(signals, widths, inputs, registers, constants, ops with their operand order)
and a small builder.  It contains none of the method's arithmetic: no op is
ever evaluated here.  Both `oracle/` and `paper_2601_18140_b200/` consume a
`Circuit`; neither imports the other.

Opcode numbers are the interchange format's (they appear, with the same
values, in `include/rtlsim.h` and in `oracle/oracle.h`, each written
independently).  The op vocabulary is the north-star list
(and/or/xor/not/add/sub/mul/shl/shr/eq/lt/mux/bits/cat); the FIRRTL reading of
each op is DESIGN.md reading R1 (§6.1 P:1269-1270 "all FIRRTL
primitive operations"; App. A P:1906 for mux).

Params per op (``param[j, 0..1]``):
  shl / shr : p0 = shift amount n
  bits      : p0 = hi, p1 = lo   (hi >= lo, hi <= 63)
  cat       : unused (w_b is the declared width of operand 1)
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

AND, OR, XOR, NOT, ADD, SUB, MUL, EQ, LT, SHL, SHR, BITS, CAT, MUX = range(14)
NUM_OPS = 14
OP_NAMES = ["and", "or", "xor", "not", "add", "sub", "mul", "eq", "lt",
            "shl", "shr", "bits", "cat", "mux"]
OP_BY_NAME = {n: i for i, n in enumerate(OP_NAMES)}

# Fixed arities; the reducible ops (and/or/xor/add/sub/mul) accept >= 2 operands
# (a left fold over the O rank, PAPER.md eq:custom_reduce P:778-796).
FOLD_OPS = (AND, OR, XOR, ADD, SUB, MUL)
FIXED_ARITY = {NOT: 1, SHL: 1, SHR: 1, BITS: 1, EQ: 2, LT: 2, CAT: 2, MUX: 3}


def arity_ok(op: int, n: int) -> bool:
    if op in FOLD_OPS:
        return n >= 2
    return FIXED_ARITY.get(op, -1) == n


@dataclass
class Circuit:
    """A synchronous circuit in canonical-id form (signal id = index)."""
    width: np.ndarray                       # u8 [n_signals], 1..64
    input_id: np.ndarray                    # u32 [n_inputs]
    reg_id: np.ndarray                      # u32 [n_regs]
    reg_next_id: np.ndarray                 # u32 [n_regs]
    reg_init: np.ndarray                    # u64 [n_regs]
    const_id: np.ndarray                    # u32 [n_consts]
    const_val: np.ndarray                   # u64 [n_consts]
    opcode: np.ndarray                      # u8 [n_ops]
    out_id: np.ndarray                      # u32 [n_ops]
    arg_off: np.ndarray                     # u32 [n_ops + 1]
    arg_id: np.ndarray                      # u32 [arg_off[-1]]
    param: np.ndarray                       # u32 [n_ops, 2]
    level: Optional[np.ndarray] = None      # u32 [n_ops] (optional; generator-exact levels)
    name: str = "circuit"
    meta: Dict = field(default_factory=dict)

    @property
    def n_signals(self) -> int:
        return int(self.width.shape[0])

    @property
    def n_inputs(self) -> int:
        return int(self.input_id.shape[0])

    @property
    def n_regs(self) -> int:
        return int(self.reg_id.shape[0])

    @property
    def n_consts(self) -> int:
        return int(self.const_id.shape[0])

    @property
    def n_ops(self) -> int:
        return int(self.opcode.shape[0])

    def normalized(self) -> "Circuit":
        """Return a copy with contiguous arrays of the interchange dtypes."""
        def a(x, dt):
            return np.array(x, dtype=dt, copy=True, order="C")
        return Circuit(
            width=a(self.width, np.uint8), input_id=a(self.input_id, np.uint32),
            reg_id=a(self.reg_id, np.uint32), reg_next_id=a(self.reg_next_id, np.uint32),
            reg_init=a(self.reg_init, np.uint64), const_id=a(self.const_id, np.uint32),
            const_val=a(self.const_val, np.uint64), opcode=a(self.opcode, np.uint8),
            out_id=a(self.out_id, np.uint32), arg_off=a(self.arg_off, np.uint32),
            arg_id=a(self.arg_id, np.uint32),
            param=a(self.param, np.uint32).reshape(-1, 2),
            level=None if self.level is None else a(self.level, np.uint32),
            name=self.name, meta=dict(self.meta))

    def permuted(self, perm: np.ndarray) -> "Circuit":
        """Rename every signal s -> perm[s] (a bijection).  Results of the
        simulation are invariant up to this renaming; used to make sure no
        consumer relies on the generator's id order."""
        perm = np.asarray(perm, dtype=np.int64)
        inv = np.empty_like(perm)
        inv[perm] = np.arange(perm.shape[0])
        c = self.normalized()
        width = c.width[inv]
        return Circuit(
            width=width, input_id=perm[c.input_id].astype(np.uint32),
            reg_id=perm[c.reg_id].astype(np.uint32),
            reg_next_id=perm[c.reg_next_id].astype(np.uint32), reg_init=c.reg_init,
            const_id=perm[c.const_id].astype(np.uint32), const_val=c.const_val,
            opcode=c.opcode, out_id=perm[c.out_id].astype(np.uint32), arg_off=c.arg_off,
            arg_id=perm[c.arg_id].astype(np.uint32), param=c.param, level=c.level,
            name=c.name + "+perm", meta=dict(c.meta)).normalized()

    def op_args(self, j: int) -> List[int]:
        return [int(x) for x in self.arg_id[self.arg_off[j]:self.arg_off[j + 1]]]

    def stats(self) -> Dict:
        ar = np.diff(self.arg_off.astype(np.int64))
        return {"n_signals": self.n_signals, "n_ops": self.n_ops, "n_inputs": self.n_inputs,
                "n_regs": self.n_regs, "n_consts": self.n_consts,
                "n_levels": int(self.level.max()) + 1 if self.level is not None and self.n_ops else None,
                "mean_arity": float(ar.mean()) if ar.size else 0.0}


class Builder:
    """Tiny netlist builder for hand-written (closed-form) circuits."""

    def __init__(self, name: str = "built"):
        self.name = name
        self.width: List[int] = []
        self.inputs: List[int] = []
        self.regs: List[int] = []
        self.reg_next: Dict[int, int] = {}
        self.reg_init: Dict[int, int] = {}
        self.consts: List[int] = []
        self.const_val: Dict[int, int] = {}
        self.ops: List[tuple] = []   # (opcode, out, args, p0, p1)

    def _sig(self, w: int) -> int:
        if not (1 <= w <= 64):
            raise ValueError(f"width {w} out of 1..64")
        self.width.append(w)
        return len(self.width) - 1

    def input(self, w: int) -> int:
        s = self._sig(w)
        self.inputs.append(s)
        return s

    def reg(self, w: int, init: int = 0) -> int:
        s = self._sig(w)
        self.regs.append(s)
        self.reg_init[s] = init
        return s

    def const(self, w: int, v: int) -> int:
        s = self._sig(w)
        self.consts.append(s)
        self.const_val[s] = v
        return s

    def op(self, name, args: Sequence[int], w: int, p0: int = 0, p1: int = 0) -> int:
        opc = OP_BY_NAME[name] if isinstance(name, str) else int(name)
        if not arity_ok(opc, len(args)):
            raise ValueError(f"bad arity {len(args)} for {OP_NAMES[opc]}")
        s = self._sig(w)
        self.ops.append((opc, s, list(args), p0, p1))
        return s

    def set_next(self, reg: int, nxt: int) -> None:
        self.reg_next[reg] = nxt

    def build(self) -> Circuit:
        missing = [r for r in self.regs if r not in self.reg_next]
        if missing:
            raise ValueError(f"registers without next: {missing}")
        arg_off = [0]
        arg_id: List[int] = []
        for (_, _, args, _, _) in self.ops:
            arg_id.extend(args)
            arg_off.append(len(arg_id))
        return Circuit(
            width=np.array(self.width, dtype=np.uint8),
            input_id=np.array(self.inputs, dtype=np.uint32),
            reg_id=np.array(self.regs, dtype=np.uint32),
            reg_next_id=np.array([self.reg_next[r] for r in self.regs], dtype=np.uint32),
            reg_init=np.array([self.reg_init[r] for r in self.regs], dtype=np.uint64),
            const_id=np.array(self.consts, dtype=np.uint32),
            const_val=np.array([self.const_val[c] for c in self.consts], dtype=np.uint64),
            opcode=np.array([o[0] for o in self.ops], dtype=np.uint8),
            out_id=np.array([o[1] for o in self.ops], dtype=np.uint32),
            arg_off=np.array(arg_off, dtype=np.uint32),
            arg_id=np.array(arg_id, dtype=np.uint32),
            param=np.array([[o[3], o[4]] for o in self.ops], dtype=np.uint32).reshape(-1, 2),
            level=None, name=self.name).normalized()
