"""Thin ctypes binding of the C ABI in include/rtlsim.h (argument marshalling
only: every simulated cycle runs in the CUDA kernels of librtlsim.so).

There is no CPU fallback: if the library is missing or has no device to run
on, calls raise.  PyTorch is used (optionally) only for device buffers and
streams.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RTLSIM_LIB") or os.path.join(_HERE, "lib", "librtlsim.so")

RS_MODE_LANES, RS_MODE_SINGLE = 0, 1
RS_LOAD_PASSES = 0x100
RS_MEM_NONE, RS_MEM_HOST, RS_MEM_DEVICE = 0, 1, 2
STATUS = {0: "RS_OK", -1: "RS_E_INVALID_ARG", -2: "RS_E_GRAPH", -3: "RS_E_CAPACITY", -4: "RS_E_OOM",
          -5: "RS_E_CUDA", -6: "RS_E_STATE", -7: "RS_E_RANGE", -8: "RS_E_UNSUPPORTED"}

# every symbol include/rtlsim.h declares
EXPORTS = ["rs_version", "rs_last_error", "rs_load_graph", "rs_graph_info_get", "rs_free_graph",
           "rs_alloc_lanes", "rs_free_lanes", "rs_lanes_bytes", "rs_set_input_seed", "rs_set_inputs",
           "rs_step_cycles", "rs_read_signals", "rs_write_registers", "rs_get_cycle", "rs_set_cycle",
           "rs_launch_count", "rs_launch_shape", "rs_lanes_kernel", "rs_repcut_stats", "rs_watch", "rs_wave_read", "rs_sync", "rs_graph_export", "rs_debug_trace",
           "rs_level_cut", "rs_ipc_handle", "rs_ipc_connect", "rs_lanes_state_bytes", "rs_lanes_bind_state",
           "rs_specialize", "rs_specialized_ptx"]
RS_DEVICE_NONE = -1
EXPORT = {"runs": (0, np.uint32), "level_run_begin": (1, np.uint32), "level_op_begin": (2, np.uint32),
          "opw": (3, np.uint32), "opk": (4, np.uint64), "coord_off": (5, np.uint32), "coord": (6, np.uint32),
          "sig_coord": (7, np.uint32), "reg_coord": (8, np.uint32), "reg_next_coord": (9, np.uint32),
          "in_coord": (10, np.uint32)}


class RtlSimError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class GraphDesc(C.Structure):
    _fields_ = [
        ("n_signals", C.c_uint32), ("width", C.c_void_p),
        ("n_inputs", C.c_uint32), ("input_id", C.c_void_p),
        ("n_regs", C.c_uint32), ("reg_id", C.c_void_p), ("reg_next_id", C.c_void_p), ("reg_init", C.c_void_p),
        ("n_consts", C.c_uint32), ("const_id", C.c_void_p), ("const_val", C.c_void_p),
        ("n_ops", C.c_uint32), ("opcode", C.c_void_p), ("out_id", C.c_void_p),
        ("arg_off", C.c_void_p), ("arg_id", C.c_void_p), ("param", C.c_void_p), ("level", C.c_void_p),
    ]


class GraphInfo(C.Structure):
    _fields_ = [
        ("mode", C.c_uint32), ("n_levels", C.c_uint32), ("n_ops", C.c_uint32), ("n_copy_ops", C.c_uint32),
        ("n_runs", C.c_uint32), ("n_coords", C.c_uint32), ("rows", C.c_uint32 * 4),
        ("state_bytes_per_lane", C.c_uint64), ("graph_device_bytes", C.c_uint64),
        ("graph_alg_bytes", C.c_uint64), ("alg_bytes_per_lane_cycle", C.c_uint64),
        ("identity_ops_naive", C.c_uint64), ("rows_bit", C.c_uint32), ("n_alias", C.c_uint32),
        ("n_folded", C.c_uint32), ("n_mux_chain", C.c_uint32),
    ]


class LaneOpts(C.Structure):
    _fields_ = [("lane0", C.c_uint64), ("lane_tile", C.c_uint32), ("threads", C.c_uint32),
                ("stage_cycles", C.c_uint32), ("cluster", C.c_uint32), ("stream", C.c_void_p),
                ("parts", C.c_uint32), ("kernel", C.c_uint32),
                ("repcut", C.c_uint32), ("repcut_global", C.c_uint32),
                ("part_world", C.c_uint32), ("part_rank", C.c_uint32), ("l2_policy", C.c_uint32),
                ("defer_state", C.c_uint32), ("op_pairs", C.c_uint32)]


_lib = None


def lib() -> C.CDLL:
    """Load librtlsim.so (building it first if the sources are newer)."""
    global _lib
    if _lib is None:
        if "RTLSIM_LIB" not in os.environ and (not os.path.exists(LIB_PATH) or
                                               os.environ.get("RTLSIM_AUTOBUILD", "1") == "1"):
            from . import build as _b
            _b.build()
        L = C.CDLL(LIB_PATH)
        vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        sig = {
            "rs_version": (C.c_char_p, []),
            "rs_last_error": (C.c_char_p, []),
            "rs_load_graph": (i32, [C.POINTER(GraphDesc), i32, u32, C.POINTER(vp)]),
            "rs_graph_info_get": (i32, [vp, C.POINTER(GraphInfo)]),
            "rs_free_graph": (None, [vp]),
            "rs_alloc_lanes": (i32, [vp, u32, C.POINTER(LaneOpts), C.POINTER(vp)]),
            "rs_free_lanes": (None, [vp]),
            "rs_lanes_bytes": (u64, [vp]),
            "rs_set_input_seed": (i32, [vp, u64]),
            "rs_set_inputs": (i32, [vp, u64, u32, vp, i32]),
            "rs_step_cycles": (i32, [vp, u32, vp, i32]),
            "rs_read_signals": (i32, [vp, vp, u32, u32, u32, vp]),
            "rs_write_registers": (i32, [vp, vp, u32, u32, u32, vp]),
            "rs_get_cycle": (i32, [vp, C.POINTER(u64)]),
            "rs_set_cycle": (i32, [vp, u64]),
            "rs_launch_count": (u64, [vp]),
            "rs_lanes_kernel": (u32, [vp]),
            "rs_repcut_stats": (i32, [vp, u32, C.POINTER(u64), C.POINTER(u32), C.POINTER(u64)]),
            "rs_watch": (i32, [vp, vp, u32, u64]),
            "rs_wave_read": (i32, [vp, vp, u64, C.POINTER(u64), C.POINTER(u64)]),
            "rs_launch_shape": (i32, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)]),
            "rs_sync": (i32, [vp]),
            "rs_graph_export": (i32, [vp, u32, vp, C.POINTER(u64)]),
            "rs_debug_trace": (i32, [vp, vp, u64]),
            "rs_level_cut": (i32, [vp, u32, vp]),
            "rs_ipc_handle": (i32, [vp, vp]),
            "rs_ipc_connect": (i32, [vp, vp]),
            "rs_lanes_state_bytes": (u64, [vp]),
            "rs_lanes_bind_state": (i32, [vp, vp, u64]),
            "rs_specialize": (i32, [vp]),
            "rs_specialized_ptx": (i32, [vp, vp, u64, C.POINTER(u64)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st: int) -> None:
    if st != 0:
        raise RtlSimError(st, lib().rs_last_error().decode())


def _arr(x, dt):
    return np.ascontiguousarray(np.asarray(x, dtype=dt))


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _dev_ptr(t) -> int:
    """Device pointer of a torch CUDA tensor (or an int address)."""
    if isinstance(t, int):
        return t
    return int(t.data_ptr())


class Graph:
    """rs_load_graph: compile a circuit (synth.Circuit or any object with the
    same arrays) into the GPU graph format on ``device``."""

    def __init__(self, circuit, device: int = 0, mode: str = "lanes", use_levels: bool = True, passes: bool = False):
        c = circuit.normalized() if hasattr(circuit, "normalized") else circuit
        self._keep = dict(
            width=_arr(c.width, np.uint8), input_id=_arr(c.input_id, np.uint32),
            reg_id=_arr(c.reg_id, np.uint32), reg_next_id=_arr(c.reg_next_id, np.uint32),
            reg_init=_arr(c.reg_init, np.uint64), const_id=_arr(c.const_id, np.uint32),
            const_val=_arr(c.const_val, np.uint64), opcode=_arr(c.opcode, np.uint8),
            out_id=_arr(c.out_id, np.uint32), arg_off=_arr(c.arg_off, np.uint32),
            arg_id=_arr(c.arg_id, np.uint32), param=_arr(c.param, np.uint32).reshape(-1),
            level=None if (getattr(c, "level", None) is None or not use_levels) else _arr(c.level, np.uint32))
        k = self._keep
        self.n_signals = int(k["width"].shape[0])
        self.n_inputs = int(k["input_id"].shape[0])
        self.n_regs = int(k["reg_id"].shape[0])
        self.n_ops = int(k["opcode"].shape[0])
        self.desc = GraphDesc(
            self.n_signals, _ptr(k["width"]), self.n_inputs, _ptr(k["input_id"]),
            self.n_regs, _ptr(k["reg_id"]), _ptr(k["reg_next_id"]), _ptr(k["reg_init"]),
            int(k["const_id"].shape[0]), _ptr(k["const_id"]), _ptr(k["const_val"]),
            self.n_ops, _ptr(k["opcode"]), _ptr(k["out_id"]), _ptr(k["arg_off"]), _ptr(k["arg_id"]),
            _ptr(k["param"]), _ptr(k["level"]))
        self.mode = RS_MODE_SINGLE if mode == "single" else RS_MODE_LANES
        self.device = device
        h = C.c_void_p()
        _check(lib().rs_load_graph(C.byref(self.desc), device, self.mode | (RS_LOAD_PASSES if passes else 0),
                                   C.byref(h)))
        self.h = h

    def info(self) -> dict:
        gi = GraphInfo()
        _check(lib().rs_graph_info_get(self.h, C.byref(gi)))
        d = {f: getattr(gi, f) for f, _ in GraphInfo._fields_}
        d["rows"] = list(gi.rows)
        return d

    def export(self, what: str) -> np.ndarray:
        """A compiled-format array (rs_graph_export); 'runs' comes back [n_runs, 5]."""
        code, dt = EXPORT[what]
        n = C.c_uint64()
        _check(lib().rs_graph_export(self.h, code, None, C.byref(n)))
        out = np.zeros(max(n.value, 1), dtype=dt)
        _check(lib().rs_graph_export(self.h, code, _ptr(out), C.byref(n)))
        out = out[:n.value]
        return out.reshape(-1, 5) if what == "runs" else out

    def repcut_stats(self, parts: int) -> dict:
        """rs_repcut_stats: replication of a parts-way RepCut plan."""
        t, m, p = C.c_uint64(), C.c_uint32(), C.c_uint64()
        _check(lib().rs_repcut_stats(self.h, parts, C.byref(t), C.byref(m), C.byref(p)))
        return {"ops_total": t.value, "max_ops": m.value, "push": p.value}

    def specialize(self) -> str:
        """rs_specialize: generate (and, on a device, load) this design's kernel 8; returns its PTX."""
        _check(lib().rs_specialize(self.h))
        n = C.c_uint64()
        _check(lib().rs_specialized_ptx(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib().rs_specialized_ptx(self.h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def level_cut(self, parts: int) -> np.ndarray:
        """rs_level_cut: level boundaries [parts + 1] of a parts-way level cut."""
        out = np.zeros(parts + 1, dtype=np.uint32)
        _check(lib().rs_level_cut(self.h, parts, _ptr(out)))
        return out

    def close(self):
        if getattr(self, "h", None):
            lib().rs_free_graph(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Lanes:
    """rs_alloc_lanes: signal state for ``n_lanes`` lanes (global ids
    lane0 .. lane0 + n_lanes - 1)."""

    def __init__(self, graph: Graph, n_lanes: int, lane0: int = 0, lane_tile: int = 0, threads: int = 0,
                 stage_cycles: int = 0, stream=None, cluster: int = 0, parts: int = 0, kernel: int = 0,
                 repcut: int = 0, repcut_global: int = 0, part_world: int = 0, part_rank: int = 0,
                 l2_policy: int = 0, state=None, op_pairs: int = 0):
        self.graph = graph
        self.n_lanes = n_lanes
        self.lane0 = lane0
        st = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        self.opts = LaneOpts(lane0, lane_tile, threads, stage_cycles, cluster, st, parts, kernel, repcut,
                             int(repcut_global), part_world, part_rank, l2_policy, 1 if state is not None else 0,
                             op_pairs)
        h = C.c_void_p()
        _check(lib().rs_alloc_lanes(graph.h, n_lanes, C.byref(self.opts), C.byref(h)))
        self.h = h
        if state is not None:
            # caller-owned signal state: "torch" -> a torch CUDA tensor allocated here; or a tensor
            self.state = self.bind_state(state)

    # ---- inputs
    def set_seed(self, seed: int) -> None:
        _check(lib().rs_set_input_seed(self.h, seed & 0xFFFFFFFFFFFFFFFF))

    def set_inputs(self, first_cycle: int, values) -> None:
        """values: [n_cycles][n_inputs][n_lanes] u64 -- numpy (host) or torch CUDA tensor."""
        if hasattr(values, "is_cuda") and values.is_cuda:
            n = int(values.shape[0])
            _check(lib().rs_set_inputs(self.h, first_cycle, n, _dev_ptr(values), 1))
            return
        v = _arr(values, np.uint64)
        n = int(v.shape[0]) if v.ndim else 0
        self._staged_keep = v
        _check(lib().rs_set_inputs(self.h, first_cycle, n, _ptr(v), 0))

    # ---- stepping
    def step(self, n_cycles: int, hashes=None):
        """hashes: None (no hash), 'host' (returns a numpy [n_cycles, n_lanes]
        u64 array), or a torch CUDA tensor / device address of
        n_cycles * n_lanes u64 (filled asynchronously)."""
        if hashes is None:
            _check(lib().rs_step_cycles(self.h, n_cycles, None, RS_MEM_NONE))
            return None
        if isinstance(hashes, str) and hashes == "host":
            out = np.zeros((n_cycles, self.n_lanes), dtype=np.uint64)
            _check(lib().rs_step_cycles(self.h, n_cycles, _ptr(out), RS_MEM_HOST))
            return out
        if isinstance(hashes, np.ndarray):
            assert hashes.dtype == np.uint64 and hashes.flags.c_contiguous and hashes.size >= n_cycles * self.n_lanes
            _check(lib().rs_step_cycles(self.h, n_cycles, _ptr(hashes), RS_MEM_HOST))
            return hashes
        _check(lib().rs_step_cycles(self.h, n_cycles, C.c_void_p(_dev_ptr(hashes)), RS_MEM_DEVICE))
        return hashes

    # ---- state access
    def read(self, ids: Sequence[int], lane_begin: int = 0, n_lanes: Optional[int] = None) -> np.ndarray:
        n = self.n_lanes - lane_begin if n_lanes is None else n_lanes
        ids_a = _arr(ids, np.uint32)
        out = np.zeros((ids_a.shape[0], n), dtype=np.uint64)
        _check(lib().rs_read_signals(self.h, _ptr(ids_a), ids_a.shape[0], lane_begin, n, _ptr(out)))
        return out

    def write_registers(self, reg_ids: Sequence[int], values, lane_begin: int = 0) -> None:
        ids_a = _arr(reg_ids, np.uint32)
        v = _arr(values, np.uint64).reshape(ids_a.shape[0], -1)
        _check(lib().rs_write_registers(self.h, _ptr(ids_a), ids_a.shape[0], lane_begin, v.shape[1], _ptr(v)))

    @property
    def cycle(self) -> int:
        c = C.c_uint64()
        _check(lib().rs_get_cycle(self.h, C.byref(c)))
        return c.value

    @cycle.setter
    def cycle(self, c: int) -> None:
        _check(lib().rs_set_cycle(self.h, c))

    def sync(self) -> None:
        _check(lib().rs_sync(self.h))

    @property
    def launches(self) -> int:
        return int(lib().rs_launch_count(self.h))

    def shape(self):
        lt, th, ct, cs = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(lib().rs_launch_shape(self.h, C.byref(lt), C.byref(th), C.byref(ct), C.byref(cs)))
        return {"lane_tile": lt.value, "threads": th.value, "ctas": ct.value, "cluster": cs.value,
                "kernel": int(lib().rs_lanes_kernel(self.h))}

    # ---- waveform capture (rs_watch / rs_wave_read)
    CHANGE = np.dtype([("cycle", np.uint64), ("lane", np.uint64), ("watch", np.uint32), ("pad_", np.uint32),
                       ("value", np.uint64)])

    def watch(self, ids: Sequence[int], capacity: int = 1 << 20) -> None:
        """Record value changes of the canonical signals ``ids`` from the next stepped cycle on."""
        ids_a = _arr(ids, np.uint32)
        _check(lib().rs_watch(self.h, _ptr(ids_a) if ids_a.size else None, ids_a.shape[0], capacity))
        self.watched = ids_a

    def wave_read(self, cap: int = 1 << 20):
        """Drain the change records: (structured array cycle/lane/watch/value, dropped count)."""
        out = np.zeros(max(cap, 1), dtype=self.CHANGE)
        n, d = C.c_uint64(), C.c_uint64()
        _check(lib().rs_wave_read(self.h, _ptr(out), cap, C.byref(n), C.byref(d)))
        return out[:n.value], d.value

    def state_bytes(self) -> int:
        return int(lib().rs_lanes_state_bytes(self.h))

    def bind_state(self, state):
        """rs_lanes_bind_state: state = "torch" (allocate a torch CUDA uint8 tensor of
        rs_lanes_state_bytes on the graph's device) or a torch CUDA tensor; returns it
        (keep it alive as long as this allocation)."""
        if isinstance(state, str) and state == "torch":
            import torch
            n = self.state_bytes()
            state = torch.empty(n + 256, dtype=torch.uint8, device=f"cuda:{self.graph.device}")
            off = (-state.data_ptr()) % 256
            state = state[off:off + n]
        _check(lib().rs_lanes_bind_state(self.h, C.c_void_p(_dev_ptr(state)),
                                         state.numel() * state.element_size()))
        return state

    # ---- level cut across processes (rs_ipc_handle / rs_ipc_connect)
    IPC_HANDLE_BYTES = 64

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(self.IPC_HANDLE_BYTES)
        _check(lib().rs_ipc_handle(self.h, buf))
        return buf.raw

    def ipc_connect(self, handles: Sequence[bytes]) -> None:
        """handles: every rank's rs_ipc_handle bytes, in rank order."""
        blob = b"".join(bytes(h) for h in handles)
        buf = C.create_string_buffer(blob, len(blob))
        _check(lib().rs_ipc_connect(self.h, buf))

    def nbytes(self) -> int:
        return int(lib().rs_lanes_bytes(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().rs_free_lanes(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
