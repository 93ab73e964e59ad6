"""CPU tests of the product library: every symbol include/rtlsim.h declares is
exported; graph validation statuses; the compiled format (RS_DEVICE_NONE,
compile only -- nothing is simulated here) decodes back to the input circuit.
"""
import os
import re
from collections import Counter

import numpy as np
import pytest

from synth import Builder, config_circuit, fuzz_circuit
from synth.circuit import MUX

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "rtlsim.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(rs):
    L = rs.lib()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(rs.EXPORTS)
    assert b"sm_100a" in L.rs_version()


def test_no_cuda_is_an_error_not_a_fallback(rs):
    """Without a GPU, loading onto a device fails with a status (no host path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c, _ = __import__("synth.closed_form", fromlist=["x"]).counter(8)
    with pytest.raises(rs.RtlSimError) as e:
        rs.Graph(c, device=0)
    assert e.value.name in ("RS_E_CUDA", "RS_E_INVALID_ARG")


def _graph(rs, c, mode="lanes"):
    return rs.Graph(c, device=rs.RS_DEVICE_NONE, mode=mode)


def test_compile_only_cannot_allocate(rs):
    c, _ = __import__("synth.closed_form", fromlist=["x"]).counter(8)
    g = _graph(rs, c)
    with pytest.raises(rs.RtlSimError) as e:
        rs.Lanes(g, 4)
    assert e.value.name == "RS_E_STATE"


def test_validation_statuses(rs):
    b = Builder()
    x = b.input(8)
    y = b.op("add", [x, x], 8)
    good = b.build()
    _graph(rs, good)

    def bad(mut, status):
        c = good.normalized()
        mut(c)
        with pytest.raises(rs.RtlSimError) as e:
            _graph(rs, c)
        assert e.value.name == status, (e.value, status)

    bad(lambda c: c.arg_id.__setitem__(0, y), "RS_E_GRAPH")                 # comb. loop
    bad(lambda c: c.out_id.__setitem__(0, x), "RS_E_GRAPH")                 # two drivers
    bad(lambda c: c.width.__setitem__(1, 0), "RS_E_GRAPH")                  # width 0
    bad(lambda c: c.width.__setitem__(1, 65), "RS_E_GRAPH")                 # width 65
    bad(lambda c: c.opcode.__setitem__(0, 3), "RS_E_GRAPH")                 # not with 2 args
    bad(lambda c: c.opcode.__setitem__(0, 99), "RS_E_GRAPH")                # unknown opcode
    bad(lambda c: c.arg_id.__setitem__(1, 77), "RS_E_GRAPH")                # id out of range
    b2 = Builder()
    z = b2.input(8)
    b2.op("bits", [z], 4, 70, 0)
    with pytest.raises(rs.RtlSimError):
        _graph(rs, b2.build())                                              # bits hi > 63
    b3 = Builder()
    z = b3.input(8)
    b3.width.append(8)                                                      # undriven signal
    b3.op("add", [z, z], 8)
    with pytest.raises(rs.RtlSimError) as e:
        _graph(rs, b3.build())
    assert e.value.name == "RS_E_GRAPH"
    c = good.normalized()                                                   # bad explicit level
    c.level = np.array([0], dtype=np.uint32)
    _graph(rs, c)
    b4 = Builder()
    z = b4.input(8)
    a = b4.op("not", [z], 8)
    b4.op("not", [a], 8)
    c4 = b4.build()
    c4.level = np.array([1, 1], dtype=np.uint32)
    with pytest.raises(rs.RtlSimError) as e:
        _graph(rs, c4)
    assert e.value.name == "RS_E_GRAPH"


def decode(rs, c, g):
    """Decode the compiled format back to (level, opcode, out id, operand ids, params)."""
    runs = g.export("runs")
    lrb = g.export("level_run_begin")
    lob = g.export("level_op_begin")
    opw = g.export("opw")
    coff = g.export("coord_off")
    coord = g.export("coord")
    sigc = g.export("sig_coord")
    n_sig = c.n_signals
    by_coord = {int(v): s for s, v in enumerate(sigc)}
    assert len(by_coord) == n_sig, "coords must be unique per signal"
    ops = []
    levels_of = {}
    for lev in range(len(lrb) - 1):
        assert lob[lev] <= lob[lev + 1]
        for r in range(lrb[lev], lrb[lev + 1]):
            ob, cnt, cb, row0, meta = (int(v) for v in runs[r])
            opc, ar, cls = meta & 0xFF, (meta >> 8) & 0xFF, (meta >> 16) & 3
            assert lob[lev] <= ob and ob + cnt <= lob[lev + 1]
            assert cb == coff[ob]
            for k in range(cnt):
                j = ob + k
                pw = int(opw[j])
                assert pw & 127 >= 1 and (pw >> 20) & 3 == cls and (pw >> 22) & 15 == opc and pw >> 26 == ar
                out_c = (cls << 30) | (row0 + k)                       # implicit S coordinate
                args_c = [int(x) for x in coord[coff[j]:coff[j + 1]]]
                assert len(args_c) == ar
                out = by_coord.get(out_c, ("copy", out_c))
                args = [by_coord.get(a, ("copy", a)) for a in args_c]
                ops.append((lev, opc, out, tuple(args), pw))
                levels_of[out_c] = lev
    return ops, levels_of, by_coord


@pytest.mark.parametrize("which", ["C1", "C2", "fuzz3", "fuzz8", "fuzz11", "paper"])
def test_format_decodes_to_input_graph(rs, which):
    """SURVEY §4.3 layer 4: the decoded graph tensor equals the input graph as a
    multiset of (opcode, out, operands in O order, params); every op reads only
    signals produced at a lower level; runs are grouped by (opcode, arity,
    width class); zero identity entries except register->source copies."""
    from synth import closed_form as cf
    if which == "paper":
        c, _ = cf.paper_example()
    elif which.startswith("fuzz"):
        c = fuzz_circuit(int(which[4:]))
    else:
        c = config_circuit(which)
    g = _graph(rs, c)
    info = g.info()
    ops, levels_of, by_coord = decode(rs, c, g)
    canon = [o for o in ops if not isinstance(o[2], tuple)]
    copies = [o for o in ops if isinstance(o[2], tuple)]
    assert len(canon) == c.n_ops and len(copies) == info["n_copy_ops"]
    want = Counter()
    for j in range(c.n_ops):
        opc = int(c.opcode[j])
        want[(opc, int(c.out_id[j]), tuple(c.op_args(j)))] += 1
    got = Counter((o[1], o[2], o[3]) for o in canon)
    assert got == want
    # params survive: w_out and shift / bits / cat parameters
    pmap = {o[2]: o[4] for o in canon}
    for j in range(c.n_ops):
        pw = pmap[int(c.out_id[j])]
        assert pw & 127 == int(c.width[c.out_id[j]])
        opc = int(c.opcode[j])
        if opc in (9, 10):
            assert (pw >> 7) & 127 == min(int(c.param[j, 0]), 64)
        if opc == 11:
            assert ((pw >> 7) & 127, (pw >> 14) & 63) == (int(c.param[j, 0]), int(c.param[j, 1]))
        if opc == 12:
            assert (pw >> 7) & 127 == int(c.width[c.op_args(j)[1]])
    # levels: operands come from strictly lower levels (or sources)
    sig_coord = g.export("sig_coord")
    for (lev, _, out, args, _) in ops:
        for a in args:
            if isinstance(a, tuple):
                continue
            ac = int(sig_coord[a])
            if ac in levels_of:
                assert levels_of[ac] < lev
    # copies only for register next edges that point at inputs / registers
    srcs = set(int(x) for x in c.input_id) | set(int(x) for x in c.reg_id)
    need = set(int(n) for n in c.reg_next_id if int(n) in srcs)
    assert len(copies) == len(need)
    rnc = g.export("reg_next_coord")
    assert all(int(x) in levels_of for x in rnc) or c.n_consts > 0


def test_format_runs_sorted_and_stats(rs):
    c = config_circuit("C3", n_ops=30000, n_levels=20, n_regs=3000)
    g = _graph(rs, c)
    info = g.info()
    runs = g.export("runs")
    lrb = g.export("level_run_begin")
    assert info["n_levels"] == 20 and info["n_runs"] == runs.shape[0]
    for lev in range(20):
        # (arity, opcode, kind, out class); kind 0 = 1-bit result of 1-bit operands, 1 = other 1-bit, 2 = wider
        keys = [((int(m) >> 8) & 0xFF, int(m) & 0xFF, (int(m) >> 18) & 3, (int(m) >> 16) & 3)
                for m in runs[lrb[lev]:lrb[lev + 1], 4]]
        assert keys == sorted(keys) and len(set(keys)) == len(keys)
    # B_alg per lane-cycle equals the SURVEY §8(d) formula recomputed here
    cls_b = lambda w: 1 if w <= 8 else 2 if w <= 16 else 4 if w <= 32 else 8
    W = [cls_b(int(w)) for w in c.width]
    B = sum(W[a] for a in c.arg_id) + sum(W[o] for o in c.out_id)
    B += sum(W[r] + W[n] for r, n in zip(c.reg_id, c.reg_next_id)) + sum(W[i] for i in c.input_id)
    assert info["alg_bytes_per_lane_cycle"] == B
    assert info["graph_alg_bytes"] == 4 * len(c.arg_id) + 4 * c.n_ops
    assert info["state_bytes_per_lane"] == sum(W)
    assert info["identity_ops_naive"] > 0
    # class-0 rows [0, rows_bit) are exactly the 1-bit signals (bit-plane layout of lane kernel 3)
    sc = g.export("sig_coord")
    nb = int(sum(1 for w in c.width if int(w) == 1))
    assert info["rows_bit"] == nb
    for s_, w in enumerate(c.width):
        co = int(sc[s_])
        assert ((co >> 30) == 0 and (co & 0x3FFFFFFF) < nb) == (int(w) == 1)


def test_identity_copy_for_register_chains(rs):
    from synth import closed_form as cf
    c, x, rs_ = cf.shift_register(5, 8)
    g = _graph(rs, c)
    assert g.info()["n_copy_ops"] == 5            # next(r0) = input, next(r_k) = register
    c2, _, _ = cf.swap(8, 1, 2)
    assert _graph(rs, c2).info()["n_copy_ops"] == 2


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_level_cut_ranges(rs, name):
    """rs_level_cut: contiguous non-empty level ranges
    covering all levels, balanced by op weight to within one level's weight."""
    c = config_circuit(name, **({"n_ops": 30000, "n_regs": 3000} if name == "C3" else {}))
    g = rs.Graph(c, device=rs.RS_DEVICE_NONE, mode="single")
    nl = g.info()["n_levels"]
    lob = g.export("level_op_begin").astype(np.int64)
    co = g.export("coord_off").astype(np.int64)
    wl = lob + co[lob]                       # cumulative weight (1 + arity) at level boundaries
    for parts in (1, 2, 3, 4, 8):
        if parts > nl:
            continue
        cut = g.level_cut(parts).astype(np.int64)
        assert cut[0] == 0 and cut[-1] == nl and np.all(np.diff(cut) >= 1)
        w = np.diff(wl[cut])
        assert w.sum() == wl[-1]
        maxlvl = np.diff(wl).max()
        assert np.all(np.abs(w - wl[-1] / parts) <= maxlvl + 1), (parts, w.tolist())
    with pytest.raises(rs.RtlSimError):
        g.level_cut(0)
    with pytest.raises(rs.RtlSimError):
        g.level_cut(9)


def test_vcd_writer_format():
    """VCD text of hand-made change records (wave.py; no GPU)."""
    from paper_2601_18140_b200 import rtlsim as rs
    from paper_2601_18140_b200.wave import changes_from_trace, vcd_string
    rec = np.zeros(5, dtype=rs.Lanes.CHANGE)
    rec["cycle"] = [0, 0, 3, 3, 1]
    rec["lane"] = [7, 7, 7, 8, 7]
    rec["watch"] = [0, 1, 1, 1, 0]
    rec["value"] = [1, 5, 6, 9, 0]
    txt = vcd_string(rec, [1, 4], lane=7, names=["clk_en", "cnt"])
    assert "$var wire 1 ! clk_en $end" in txt and '$var wire 4 " cnt $end' in txt
    body = txt.split("$enddefinitions $end\n")[1]
    assert body == '#0\n1!\nb101 "\n#1\n0!\n#3\nb110 "\n'
    # change-set semantics: first cycle always, then only differences
    tr = np.array([[[1, 2]], [[1, 3]], [[4, 3]]], dtype=np.uint64)   # [cycle][watch][lane]
    assert changes_from_trace(tr, 10, [0, 1]) == {(10, 0, 0, 1), (10, 1, 0, 2), (11, 1, 0, 3), (12, 0, 0, 4)}


def test_repcut_plan_stats(rs):
    """rs_repcut_stats (App. C, Cascade 2):
    one partition holds every op once and pushes nothing; a multi-core design
    with no cross-core edges, cut at its core boundaries, replicates nothing
    and pushes nothing; coupling through registers adds pushes; replication is
    bounded by P copies of the graph."""
    from synth import multicore_circuit
    c = multicore_circuit(4, 600, 10, 60, 4, cross_p=0.0, seed=5)
    g = rs.Graph(c, device=rs.RS_DEVICE_NONE, mode="single")
    n = g.info()
    total = n["n_ops"] + n["n_copy_ops"]
    one = g.repcut_stats(1)
    assert one == {"ops_total": total, "max_ops": total, "push": 0}
    four = g.repcut_stats(4)
    assert four["ops_total"] == total and four["push"] == 0
    assert four["max_ops"] < total
    two = g.repcut_stats(2)
    assert two["ops_total"] == total and two["push"] == 0
    cc = multicore_circuit(4, 600, 10, 60, 4, cross_p=0.02, seed=5)
    gc = rs.Graph(cc, device=rs.RS_DEVICE_NONE, mode="single")
    tc = gc.info()["n_ops"] + gc.info()["n_copy_ops"]
    for P in (2, 3, 4, 7):
        st = gc.repcut_stats(P)
        assert tc <= st["ops_total"] <= P * tc
        assert -(-st["ops_total"] // P) <= st["max_ops"] <= tc
        assert st["push"] > 0
    with pytest.raises(rs.RtlSimError):
        gc.repcut_stats(0)
    with pytest.raises(rs.RtlSimError):
        gc.repcut_stats(256)


def test_header_is_plain_c():
    """include/rtlsim.h is a C ABI: it compiles as C99 (no C++ or torch types),
    and a C program can link the library's entry points."""
    import shutil
    import subprocess
    import tempfile
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no C compiler")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([gcc, "-fsyntax-only", "-std=c99", "-Wall", "-Werror", "-x", "c",
                        os.path.join(root, "include", "rtlsim.h")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    src = """#include "rtlsim.h"
int main(void) { rs_graph* g = 0; rs_graph_desc d = {0};
  rs_status s = rs_load_graph(&d, RS_DEVICE_NONE, RS_MODE_LANES, &g);
  return s == RS_OK ? 0 : (rs_last_error() ? 0 : 1); }"""
    lib = os.path.join(root, "paper_2601_18140_b200", "lib")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        r = subprocess.run([gcc, "-std=c99", "-I", os.path.join(root, "include"), c, "-L", lib, "-lrtlsim",
                            "-Wl,-rpath," + lib, "-o", os.path.join(d, "t")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_repcut_partition_recovers_shuffled_cores(rs):
    """RepCut register partition (compiler.cpp cone_cluster_partition, reading R20): with
    the registers listed in a random order, contiguous index blocks replicate ~10x
    (2.0M ops for 200k at P = 16); grouping registers by the connected component of their
    combinational logic finds the 16 cores again -- replication-free, balanced."""
    import dataclasses
    from synth import multicore_circuit
    c = multicore_circuit()
    perm = np.random.default_rng(0).permutation(c.n_regs)
    cs = dataclasses.replace(c, reg_id=c.reg_id[perm], reg_next_id=c.reg_next_id[perm], reg_init=c.reg_init[perm])
    for circ in (c, cs):
        g = rs.Graph(circ, device=rs.RS_DEVICE_NONE, mode="single")
        st = g.repcut_stats(16)
        assert st["ops_total"] == g.info()["n_ops"]
        assert st["max_ops"] <= 12_600
    # a random single core has one logic component: the contiguous blocks stay
    g5 = rs.Graph(config_circuit("C3", n_ops=20000, n_levels=30, n_regs=2000), device=rs.RS_DEVICE_NONE, mode="single")
    st = g5.repcut_stats(4)
    assert st["ops_total"] >= g5.info()["n_ops"]
