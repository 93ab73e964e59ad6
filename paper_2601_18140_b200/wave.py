"""Waveform output (§6.2, where
the DMI writes waveforms of the simulated design).

The change records come from the step kernel (``Lanes.watch`` /
``Lanes.wave_read``, C ABI ``rs_watch`` / ``rs_wave_read``): one record per
(cycle, lane, watched signal) whose value changed.  This module only formats
them -- host-side text output, off the simulation path.
"""
from __future__ import annotations

import io
from typing import Optional, Sequence, TextIO, Union

import numpy as np

_ID_CHARS = "".join(chr(c) for c in range(33, 127))


def _vcd_id(i: int) -> str:
    s = ""
    while True:
        s += _ID_CHARS[i % len(_ID_CHARS)]
        i //= len(_ID_CHARS)
        if i == 0:
            return s


def write_vcd(out: Union[str, TextIO], records: np.ndarray, widths: Sequence[int], lane: int,
              names: Optional[Sequence[str]] = None, module: str = "top") -> None:
    """Write the records of one lane as a VCD file (1 time unit = 1 cycle).

    records: structured array with fields cycle, lane, watch, value (as
    returned by ``Lanes.wave_read``); widths[i] / names[i] describe watch i."""
    if isinstance(out, str):
        with open(out, "w") as f:
            return write_vcd(f, records, widths, lane, names, module)
    n = len(widths)
    names = list(names) if names is not None else [f"s{i}" for i in range(n)]
    r = records[records["lane"] == np.uint64(lane)]
    r = r[np.lexsort((r["watch"], r["cycle"]))]
    out.write("$timescale 1ns $end\n")
    out.write(f"$scope module {module} $end\n")
    for i in range(n):
        out.write(f"$var wire {int(widths[i])} {_vcd_id(i)} {names[i]} $end\n")
    out.write("$upscope $end\n$enddefinitions $end\n")
    cur = None
    for rec in r:
        c = int(rec["cycle"])
        if c != cur:
            out.write(f"#{c}\n")
            cur = c
        w, v, i = int(widths[int(rec["watch"])]), int(rec["value"]), int(rec["watch"])
        if w == 1:
            out.write(f"{v & 1}{_vcd_id(i)}\n")
        else:
            out.write(f"b{v:b} {_vcd_id(i)}\n")


def vcd_string(records: np.ndarray, widths: Sequence[int], lane: int, names: Optional[Sequence[str]] = None) -> str:
    buf = io.StringIO()
    write_vcd(buf, records, widths, lane, names)
    return buf.getvalue()


def changes_from_trace(trace: np.ndarray, first_cycle: int, lanes: Sequence[int]) -> set:
    """The change-record set a per-cycle value trace [n_cycles][n_watch][n_lanes]
    implies: every (signal, lane) at the first cycle, then whenever the value
    differs from the previous cycle.  Elements: (cycle, lane, watch, value)."""
    out = set()
    nc, nw, nl = trace.shape
    for c in range(nc):
        for w in range(nw):
            for j in range(nl):
                v = int(trace[c, w, j])
                if c == 0 or v != int(trace[c - 1, w, j]):
                    out.add((first_cycle + c, int(lanes[j]), w, v))
    return out
