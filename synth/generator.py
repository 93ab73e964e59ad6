"""Seeded synthetic circuits shaped like BASELINE.json's configs C1-C5.

The paper measures on Chipyard designs (§7) that are not
available; these seeded random levelized circuits stand in for them
(DESIGN.md §"Inputs").  The recipe is SURVEY.md §8(d) "Generator":

* ``N/L`` ops per level (remainder to the first levels); level -1 = sources.
* each op draws an opcode from the config's mix, then its width;
* the anchor operand (operand 0; operand 1 for mux) is uniform over level
  l-1, so ASAP levels are exact; every other operand is, with p=0.7, uniform
  over levels [l-3, l-1] (clamped, sources included) and with p=0.3 uniform
  over all signals of level < l;
* a mux selector is drawn from the 1-bit signals of the same pool when any
  exist;
* shl n ~ U[0, w_out-1]; shr n ~ U[0, w(x0)-1]; bits lo ~ U[0, w(x0)-1],
  hi = min(lo + w_out - 1, 63); cat w_b = w(x1); not w_out = w(x0);
  eq / lt w_out = 1 (FIRRTL);
* registers: width from the distribution, next uniform over op outputs, init 0;
* inputs: width from the distribution (stimulus: ``synth.stimulus``).

Nothing here evaluates an op: the module only draws structure.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Optional

import numpy as np

from .circuit import (ADD, AND, BITS, CAT, EQ, LT, MUL, MUX, NOT, OR, SHL, SHR,
                      SUB, XOR, NUM_OPS, Circuit, FOLD_OPS)


def _mix(weights: Dict[int, float]) -> np.ndarray:
    p = np.zeros(NUM_OPS, dtype=np.float64)
    for k, v in weights.items():
        p[k] = v
    return p / p.sum()


MIX_C1 = _mix({o: 1.0 for o in (AND, OR, XOR, NOT, ADD, SUB, EQ, LT, MUX, SHL, SHR, BITS, CAT)})
MIX_ALL = _mix({o: 1.0 for o in range(NUM_OPS)})
_C3_REST = (AND, OR, XOR, NOT, EQ, LT, SHL, SHR, BITS, CAT, MUL)
MIX_C3 = _mix({MUX: 0.10, ADD: 0.075, SUB: 0.075, **{o: 0.75 / len(_C3_REST) for o in _C3_REST}})


def sample_width(rng: np.random.Generator, dist: str, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    if dist == "u1_16":
        return rng.integers(1, 17, size=n)
    if dist == "c2":          # 60% U[1,8], 40% U[9,64]
        lo = rng.integers(1, 9, size=n)
        hi = rng.integers(9, 65, size=n)
        return np.where(rng.random(n) < 0.6, lo, hi)
    if dist == "c3":          # 50% 1-bit, 30% U[2,32], 20% 64-bit
        u = rng.random(n)
        mid = rng.integers(2, 33, size=n)
        return np.where(u < 0.5, 1, np.where(u < 0.8, mid, 64))
    if dist == "u1_64":
        return rng.integers(1, 65, size=n)
    raise ValueError(dist)


@dataclass(frozen=True)
class GenConfig:
    name: str
    n_ops: int
    n_levels: int
    n_regs: int
    n_inputs: int
    mix: tuple
    width_dist: str
    p3: float            # probability of a 3-operand fold for and/or/xor/add
    struct_seed: int
    stim_seed: int
    lanes: int
    cycles: int
    n_consts: int = 0
    reg_next_source_p: float = 0.0   # fuzz only: next(r) drawn from sources


def _cfg(name, n_ops, n_levels, n_regs, n_inputs, mix, wd, p3, ss, st, lanes, cycles):
    return GenConfig(name, n_ops, n_levels, n_regs, n_inputs, tuple(mix), wd, p3, ss, st, lanes, cycles)


# BASELINE.json configs (SURVEY.md §8(d) per-config table).
CONFIGS: Dict[str, GenConfig] = {
    "C1": _cfg("C1", 256, 12, 32, 8, MIX_C1, "u1_16", 0.0, 101, 201, 1, 1000),
    "C2": _cfg("C2", 20_000, 40, 2_000, 64, MIX_ALL, "c2", 0.1, 102, 202, 1024, 10_000),
    "C3": _cfg("C3", 150_000, 80, 20_000, 128, MIX_C3, "c3", 0.0, 103, 203, 4096, 10_000),
    "C4": _cfg("C4", 2_000_000, 150, 250_000, 512, MIX_C3, "c3", 0.0, 104, 204, 8192, 2_000),
    "C5": _cfg("C5", 2_000_000, 150, 250_000, 512, MIX_C3, "c3", 0.0, 105, 205, 1, 100_000),
}


def generate(cfg: GenConfig, n_ops: Optional[int] = None, n_levels: Optional[int] = None,
             n_regs: Optional[int] = None, n_inputs: Optional[int] = None,
             seed: Optional[int] = None, permute: bool = False) -> Circuit:
    """Draw the circuit for ``cfg`` (sizes overridable for scaled-down parity cases)."""
    N = cfg.n_ops if n_ops is None else n_ops
    NL = cfg.n_levels if n_levels is None else n_levels
    R = cfg.n_regs if n_regs is None else n_regs
    I = cfg.n_inputs if n_inputs is None else n_inputs
    K = cfg.n_consts
    if N > 0 and I + R + K == 0:
        I = 1                           # level 0 needs at least one source
    seed = cfg.struct_seed if seed is None else seed
    rng = np.random.default_rng(seed)
    mix = np.asarray(cfg.mix, dtype=np.float64)
    NL = max(1, min(NL, N)) if N > 0 else 0

    S0 = I + R + K                      # sources: [inputs][regs][consts]
    n_sig = S0 + N
    width = np.zeros(n_sig, dtype=np.int64)
    width[:S0] = sample_width(rng, cfg.width_dist, S0)
    # level l occupies ids [start[l], start[l+1]); start[0] = 0 is "level -1" (sources)
    per = [N // NL + (1 if l < N % NL else 0) for l in range(NL)] if NL else []
    start = np.zeros(NL + 2, dtype=np.int64)
    start[1] = S0
    for l in range(NL):
        start[l + 2] = start[l + 1] + per[l]

    opcode = np.zeros(N, dtype=np.int64)
    arity = np.zeros(N, dtype=np.int64)
    args = np.zeros((N, 3), dtype=np.int64)
    params = np.zeros((N, 2), dtype=np.int64)
    level = np.zeros(N, dtype=np.int64)

    ones = np.zeros(n_sig, dtype=np.int64)  # sorted ids of 1-bit signals, fill pointer
    n_ones = 0
    src1 = np.nonzero(width[:S0] == 1)[0]
    ones[:src1.size] = src1
    n_ones = src1.size

    def draw_pool(n, l, rng):
        """Non-anchor operand draw: 70% from levels [l-3, l-1], 30% from all < l."""
        hi = start[l + 1]
        near_lo = start[max(l - 3, -1) + 1]
        near = rng.random(n) < 0.7
        lo = np.where(near, near_lo, 0)
        return lo, hi, (lo + np.floor(rng.random(n) * (hi - lo)).astype(np.int64))

    for l in range(NL):
        n = per[l]
        if n == 0:
            continue
        base = start[l + 1] - S0          # op index of the level's first op
        idx = slice(base, base + n)
        opc = rng.choice(NUM_OPS, size=n, p=mix)
        w = sample_width(rng, cfg.width_dist, n)
        ar = np.ones(n, dtype=np.int64) * 2
        ar[np.isin(opc, (NOT, SHL, SHR, BITS))] = 1
        ar[opc == MUX] = 3
        if cfg.p3 > 0:
            f3 = np.isin(opc, (AND, OR, XOR, ADD)) & (rng.random(n) < cfg.p3)
            ar[f3] = 3
        prev_lo, prev_hi = start[l], start[l + 1]           # level l-1
        anchor = prev_lo + np.floor(rng.random(n) * (prev_hi - prev_lo)).astype(np.int64)
        a = np.zeros((n, 3), dtype=np.int64)
        _, _, o1 = draw_pool(n, l, rng)
        _, _, o2 = draw_pool(n, l, rng)
        a[:, 0] = anchor
        a[:, 1] = o1
        a[:, 2] = o2
        # mux: anchor is operand 1 (value), selector (operand 0) prefers 1-bit signals
        m = np.nonzero(opc == MUX)[0]
        if m.size:
            slo, shi, sel_any = draw_pool(m.size, l, rng)
            i0 = np.searchsorted(ones[:n_ones], slo)
            i1 = np.searchsorted(ones[:n_ones], shi)
            cnt = i1 - i0
            pick = i0 + np.floor(rng.random(m.size) * np.maximum(cnt, 1)).astype(np.int64)
            pick = np.minimum(pick, max(n_ones - 1, 0))
            sel = np.where(cnt > 0, ones[pick] if n_ones else sel_any, sel_any)
            a[m, 1] = anchor[m]
            a[m, 0] = sel
        # widths that depend on operands
        w = np.where(np.isin(opc, (EQ, LT)), 1, w)
        w0 = width[a[:, 0]]
        w = np.where(opc == NOT, w0, w)
        p = np.zeros((n, 2), dtype=np.int64)
        sh = opc == SHL
        p[sh, 0] = np.floor(rng.random(sh.sum()) * w[sh]).astype(np.int64)
        sr = opc == SHR
        p[sr, 0] = np.floor(rng.random(sr.sum()) * w0[sr]).astype(np.int64)
        bt = opc == BITS
        lo_b = np.floor(rng.random(bt.sum()) * w0[bt]).astype(np.int64)
        p[bt, 1] = lo_b
        p[bt, 0] = np.minimum(lo_b + w[bt] - 1, 63)
        opcode[idx] = opc
        arity[idx] = ar
        args[idx] = a
        params[idx] = p
        level[idx] = l
        ids = np.arange(start[l + 1], start[l + 2])
        width[ids] = w
        new1 = ids[w == 1]
        ones[n_ones:n_ones + new1.size] = new1
        n_ones += new1.size

    # registers: next uniform over op outputs (or, for fuzz, sometimes a source)
    reg_ids = np.arange(I, I + R)
    if N > 0:
        nxt = S0 + rng.integers(0, N, size=R)
    else:
        nxt = rng.integers(0, max(S0, 1), size=R)
    if cfg.reg_next_source_p > 0 and S0 > 0:
        src = rng.random(R) < cfg.reg_next_source_p
        nxt = np.where(src, rng.integers(0, S0, size=R), nxt)
    reg_init = np.zeros(R, dtype=np.uint64)
    const_ids = np.arange(I + R, I + R + K)
    const_val = np.zeros(K, dtype=np.uint64)
    if K:
        raw = rng.integers(0, 2**63, size=K, dtype=np.int64).astype(np.uint64) * np.uint64(2) \
            + rng.integers(0, 2, size=K).astype(np.uint64)
        wk = width[const_ids].astype(np.uint64)
        mask = np.where(wk >= 64, np.uint64(0xFFFFFFFFFFFFFFFF),
                        (np.uint64(1) << np.minimum(wk, 63)) - np.uint64(1))
        const_val = raw & mask
        if cfg.reg_next_source_p > 0:     # fuzz: also exercise unmasked reg init
            reg_init = rng.integers(0, 2**63, size=R, dtype=np.int64).astype(np.uint64)

    arg_off = np.zeros(N + 1, dtype=np.int64)
    arg_off[1:] = np.cumsum(arity)
    mask3 = np.arange(3)[None, :] < arity[:, None]
    arg_id = args[mask3]
    c = Circuit(
        width=width.astype(np.uint8), input_id=np.arange(0, I, dtype=np.uint32),
        reg_id=reg_ids.astype(np.uint32), reg_next_id=nxt.astype(np.uint32), reg_init=reg_init,
        const_id=const_ids.astype(np.uint32), const_val=const_val,
        opcode=opcode.astype(np.uint8), out_id=np.arange(S0, S0 + N, dtype=np.uint32),
        arg_off=arg_off.astype(np.uint32), arg_id=arg_id.astype(np.uint32),
        param=params.astype(np.uint32), level=level.astype(np.uint32),
        name=cfg.name, meta={"struct_seed": seed, "stim_seed": cfg.stim_seed,
                             "lanes": cfg.lanes, "cycles": cfg.cycles}).normalized()
    if permute:
        prng = np.random.default_rng(seed ^ 0xA5A5)
        c = c.permuted(prng.permutation(c.n_signals))
    return c


def config_circuit(name: str, **kw) -> Circuit:
    return generate(CONFIGS[name], **kw)


def fuzz_circuit(seed: int) -> Circuit:
    """Fuzz corpus member (<= 200 ops, <= 8 levels, widths <= 64;
    SPEC.md S:405).  Exercises constants, register-to-source next edges, wide
    folds and a random canonical-id permutation."""
    rng = np.random.default_rng(10_000 + seed)
    n_ops = int(rng.integers(0, 201))
    n_levels = int(rng.integers(1, 9))
    wd = ["u1_16", "c2", "c3", "u1_64"][seed % 4]
    cfg = GenConfig(f"fuzz{seed}", n_ops, n_levels, int(rng.integers(0, 24)),
                    int(rng.integers(0, 9)), tuple(MIX_ALL), wd, 0.1, 10_000 + seed,
                    20_000 + seed, 1, 100, n_consts=int(rng.integers(0, 4)),
                    reg_next_source_p=0.2)
    return generate(cfg, permute=bool(seed % 2))


def multicore_circuit(n_cores: int = 16, ops_per_core: int = 12_500, n_levels: int = 60,
                      regs_per_core: int = 1_250, inputs_per_core: int = 8, cross_p: float = 0.01,
                      seed: int = 106, base: str = "C3") -> Circuit:
    """A partition-friendly single-design circuit for the RepCut path (SURVEY.md
    §8(f) NEXT-2; App. C, Cascade 2): ``n_cores`` independent
    ``base``-shaped random cores, like the paper's multi-core RocketChip
    configurations (r1..r24), coupled only through registers: each
    non-anchor operand is, with probability ``cross_p``, replaced by a register
    of another core.  Cores are laid out one after the other (their inputs,
    registers and ops keep per-core contiguous ids), so a register partition by
    contiguous index ranges follows the cores and needs no op replication."""
    cfg = CONFIGS[base]
    parts = [generate(cfg, n_ops=ops_per_core, n_levels=n_levels, n_regs=regs_per_core,
                      n_inputs=inputs_per_core, seed=seed * 1000 + k) for k in range(n_cores)]
    off = np.cumsum([0] + [p.n_signals for p in parts])
    width = np.concatenate([p.width for p in parts])
    cat = lambda f: np.concatenate([getattr(p, f).astype(np.int64) + off[k] for k, p in enumerate(parts)])
    input_id, reg_id, reg_next_id = cat("input_id"), cat("reg_id"), cat("reg_next_id")
    out_id, arg_id = cat("out_id"), cat("arg_id")
    const_id = cat("const_id") if sum(p.n_consts for p in parts) else np.zeros(0, np.int64)
    arg_off = np.zeros(1, dtype=np.int64)
    for p in parts:
        arg_off = np.concatenate([arg_off, arg_off[-1] + p.arg_off[1:].astype(np.int64)])
    opcode = np.concatenate([p.opcode for p in parts])
    param = np.concatenate([p.param for p in parts])
    level = np.concatenate([p.level for p in parts])
    rng = np.random.default_rng(seed)
    # cross-core coupling through registers: operand o >= 1 of an op (never the
    # anchor, so the levels stay exact) becomes a register of another core
    core_of_op = np.repeat(np.arange(n_cores), [p.n_ops for p in parts])
    ar = np.diff(arg_off)
    pos_in_op = np.arange(arg_id.shape[0]) - np.repeat(arg_off[:-1], ar)
    anchor = np.where(np.repeat(opcode == MUX, ar), 1, 0)      # per operand: the op's anchor position
    cand = np.nonzero((pos_in_op != anchor) & (rng.random(arg_id.shape[0]) < cross_p))[0]
    if n_cores > 1 and cand.size:
        core = np.repeat(core_of_op, ar)[cand]
        other = (core + rng.integers(1, n_cores, size=cand.size)) % n_cores
        pick = rng.integers(0, regs_per_core, size=cand.size)
        arg_id[cand] = reg_id[other * regs_per_core + pick]
    return Circuit(
        width=width.astype(np.uint8), input_id=input_id.astype(np.uint32), reg_id=reg_id.astype(np.uint32),
        reg_next_id=reg_next_id.astype(np.uint32), reg_init=np.concatenate([p.reg_init for p in parts]),
        const_id=const_id.astype(np.uint32), const_val=np.concatenate([p.const_val for p in parts]),
        opcode=opcode, out_id=out_id.astype(np.uint32), arg_off=arg_off.astype(np.uint32),
        arg_id=arg_id.astype(np.uint32), param=param, level=level, name=f"multicore{n_cores}x{ops_per_core}",
        meta={"struct_seed": seed, "stim_seed": 206, "lanes": 1, "cycles": 10_000}).normalized()
