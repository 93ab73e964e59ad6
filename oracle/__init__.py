"""CPU oracle for the RTeAAL Sim hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2601_18140_b200``) never imports it and shares no code
with it.  See ``oracle/oracle.h`` for what it computes and the PAPER.md
passages it follows; DESIGN.md §"Oracle" lists the readings it takes.

Pins (tests/test_oracle_*.py): paper worked example, closed
forms (counter, accumulator = the paper's prefix sum P:401-415, ripple adder,
LFSR period, shift register, swap), per-op exhaustive checks against a
big-integer definition, exhaustive truth tables, the published splitmix64
test vector.  The random C2-C5 circuits have no closed form: their parity
rests on this oracle (DESIGN.md "parity unpinned" note).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC",
                               src, "-o", _LIB])
    return _LIB


class _Circ(C.Structure):
    _fields_ = [
        ("n_signals", C.c_uint32), ("width", C.c_void_p),
        ("n_inputs", C.c_uint32), ("input_id", C.c_void_p),
        ("n_regs", C.c_uint32), ("reg_id", C.c_void_p), ("reg_next_id", C.c_void_p),
        ("reg_init", C.c_void_p),
        ("n_consts", C.c_uint32), ("const_id", C.c_void_p), ("const_val", C.c_void_p),
        ("n_ops", C.c_uint32), ("opcode", C.c_void_p), ("out_id", C.c_void_p),
        ("arg_off", C.c_void_p), ("arg_id", C.c_void_p), ("param", C.c_void_p),
    ]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            u64, u32 = C.c_uint64, C.c_uint32
            L.orc_mask.restype = u64
            L.orc_mask.argtypes = [u32]
            L.orc_splitmix_next.restype = u64
            L.orc_splitmix_next.argtypes = [u64]
            L.orc_stimulus.restype = u64
            L.orc_stimulus.argtypes = [u64, u64, u64, u64]
            L.orc_hash_weight.restype = u64
            L.orc_hash_weight.argtypes = [u64]
            L.orc_apply_op.restype = u64
            L.orc_apply_op.argtypes = [u32, u32, C.c_void_p, u32, u32, u32, u32, C.POINTER(C.c_int)]
            L.orc_topo_order.restype = C.c_int
            L.orc_topo_order.argtypes = [C.POINTER(_Circ), C.c_void_p]
            L.orc_simulate.restype = C.c_int
            L.orc_simulate.argtypes = [C.POINTER(_Circ), u64, C.c_void_p, C.c_void_p, u64, u32,
                                       u64, u32, C.c_void_p, C.c_void_p, u32, C.c_void_p, C.c_void_p]
            _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


class _Bound:
    """Keeps the numpy arrays alive while the C struct points at them."""

    def __init__(self, circ):
        c = circ.normalized()
        self.c = c
        self.s = _Circ(c.n_signals, _p(c.width), c.n_inputs, _p(c.input_id), c.n_regs,
                       _p(c.reg_id), _p(c.reg_next_id), _p(c.reg_init), c.n_consts,
                       _p(c.const_id), _p(c.const_val), c.n_ops, _p(c.opcode), _p(c.out_id),
                       _p(c.arg_off), _p(c.arg_id), _p(c.param))


def mask(w: int) -> int:
    return int(lib().orc_mask(w))


def splitmix_next(x: int) -> int:
    return int(lib().orc_splitmix_next(x & 0xFFFFFFFFFFFFFFFF))


def stimulus(seed: int, k: int, c: int, lane: int) -> int:
    return int(lib().orc_stimulus(seed, k, c, lane))


def hash_weight(s: int) -> int:
    return int(lib().orc_hash_weight(s))


def apply_op(opcode: int, xs: Sequence[int], w_out: int, p0: int = 0, p1: int = 0,
             wb: int = 0) -> int:
    arr = np.ascontiguousarray(np.array([int(x) for x in xs] or [0], dtype=np.uint64))
    ok = C.c_int(0)
    r = lib().orc_apply_op(opcode, len(xs), arr.ctypes.data, p0, p1, wb, w_out, C.byref(ok))
    if not ok.value:
        raise ValueError("bad op")
    return int(r)


def topo_order(circ) -> np.ndarray:
    b = _Bound(circ)
    order = np.zeros(max(b.c.n_ops, 1), dtype=np.uint32)
    rc = lib().orc_topo_order(C.byref(b.s), order.ctypes.data)
    if rc != 0:
        raise ValueError(f"orc_topo_order failed: {rc}")
    return order[:b.c.n_ops]


class OracleResult:
    def __init__(self, hashes, trace, final_state):
        self.hashes = hashes            # [n_cycles, n_lanes] u64
        self.trace = trace              # [n_cycles, n_watch, n_lanes] u64
        self.final_state = final_state  # [n_signals, n_lanes] u64


def simulate(circ, n_cycles: int, seed: int = 0, lane0: int = 0, n_lanes: int = 1,
             cycle0: int = 0, staged: Optional[np.ndarray] = None,
             reg_state0: Optional[np.ndarray] = None, hashes: bool = True,
             watch: Optional[Sequence[int]] = None, final: bool = False,
             threads: int = 1, lanes: Optional[Sequence[int]] = None) -> OracleResult:
    """Run the oracle.  ``lanes`` (optional) is an explicit list of global lane
    ids to simulate instead of the range [lane0, lane0+n_lanes) (used for
    sampled parity at full size); staged/reg_state0 are then indexed by
    position in that list."""
    b = _Bound(circ)
    L = lib()
    if lanes is not None:
        lane_list = [int(x) for x in lanes]
    else:
        lane_list = None
    nl = len(lane_list) if lane_list is not None else n_lanes
    watch_a = None if watch is None else np.ascontiguousarray(np.asarray(watch, dtype=np.uint32))
    nw = 0 if watch_a is None else watch_a.shape[0]
    H = np.zeros((n_cycles, nl), dtype=np.uint64) if hashes else None
    T = np.zeros((n_cycles, nw, nl), dtype=np.uint64) if nw else None
    F = np.zeros((b.c.n_signals, nl), dtype=np.uint64) if final else None
    if staged is not None:
        staged = np.ascontiguousarray(np.asarray(staged, dtype=np.uint64).reshape(n_cycles, b.c.n_inputs, nl))
    if reg_state0 is not None:
        reg_state0 = np.ascontiguousarray(np.asarray(reg_state0, dtype=np.uint64).reshape(b.c.n_regs, nl))

    # chunks of consecutive positions that map to consecutive global lanes
    if lane_list is None:
        chunks = [(0, nl, lane0)]
    else:
        chunks = []
        i = 0
        while i < nl:
            j = i + 1
            while j < nl and lane_list[j] == lane_list[j - 1] + 1:
                j += 1
            chunks.append((i, j, lane_list[i]))
            i = j
    # split big chunks for threading
    work = []
    per = max(1, -(-nl // max(1, threads)))
    for (a, e, g0) in chunks:
        s = a
        while s < e:
            t = min(e, s + per)
            work.append((s, t, g0 + (s - a)))
            s = t

    def run(item):
        a, e, g0 = item
        n = e - a
        h = np.zeros((n_cycles, n), dtype=np.uint64) if hashes else None
        t = np.zeros((n_cycles, nw, n), dtype=np.uint64) if nw else None
        f = np.zeros((b.c.n_signals, n), dtype=np.uint64) if final else None
        st = None if staged is None else np.ascontiguousarray(staged[:, :, a:e])
        r0 = None if reg_state0 is None else np.ascontiguousarray(reg_state0[:, a:e])
        rc = L.orc_simulate(C.byref(b.s), seed, _p(st), _p(r0), cycle0, n_cycles, g0, n,
                            _p(h), _p(watch_a), nw, _p(t), _p(f))
        if rc != 0:
            raise ValueError(f"orc_simulate failed: {rc}")
        return item, h, t, f

    if threads > 1 and len(work) > 1:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            results = list(ex.map(run, work))
    else:
        results = [run(w) for w in work]
    for (a, e, _), h, t, f in results:
        if H is not None:
            H[:, a:e] = h
        if T is not None:
            T[:, :, a:e] = t
        if F is not None:
            F[:, a:e] = f
    return OracleResult(H, T, F)
