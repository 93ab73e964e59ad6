"""Kernel 8: the design's own specialised kernel (rs_specialize; SURVEY.md §8(f) NEXT-4,
the GPU analog of the paper's SU mode, §5.2, Tables 4-6).

CPU tests: the generated PTX assembles with ptxas for sm_100a (no GPU needed) and the op
cap is enforced.  GPU tests: per-cycle hashes and the full final state against the oracle,
bit for bit -- single lane (one warp, stimulus spread over its threads) and lanes (one
thread per lane, several tiles, lane0 offset), seeded and staged inputs, several launches
(registers carried through the state), graph passes on and off, and the op-semantics edge
circuit with its corner values.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle
from synth import CONFIGS, config_circuit, fuzz_circuit
from synth.edge import edge_circuit, edge_values, pass_circuit

PTXAS = shutil.which("ptxas") or "/usr/local/cuda/bin/ptxas"


def _ptxas(tmp_path, ptx):
    src = tmp_path / "k8.ptx"
    src.write_text(ptx)
    return subprocess.run([PTXAS, "-arch=sm_100a", str(src), "-o", str(tmp_path / "k8.cubin")],
                          capture_output=True, text=True, timeout=300)


@pytest.mark.skipif(not os.path.exists(PTXAS), reason="ptxas not in this image")
@pytest.mark.parametrize("name", ["C1", "edge", "fuzz", "pass"])
def test_specialized_ptx_assembles(rs, tmp_path, name):
    c, mode = {"C1": (config_circuit("C1"), "single"), "edge": (edge_circuit(0), "lanes"),
               "fuzz": (fuzz_circuit(3), "lanes"), "pass": (pass_circuit(1), "single")}[name]
    g = rs.Graph(c, device=rs.RS_DEVICE_NONE, mode=mode, passes=(name == "pass"))
    ptx = g.specialize()
    assert ".entry rs_su" in ptx and ".target sm_100a" in ptx
    r = _ptxas(tmp_path, ptx)
    assert r.returncode == 0, r.stderr[-2000:]


def test_specialize_op_cap(rs):
    g = rs.Graph(config_circuit("C2"), device=rs.RS_DEVICE_NONE)
    with pytest.raises(rs.RtlSimError, match="capped"):
        g.specialize()


def _check(rs, c, n, nl, mode="lanes", passes=False, staged=None, seed=5, chunks=(3,), **kw):
    g = rs.Graph(c, device=0, mode=mode, passes=passes)
    L = rs.Lanes(g, nl, kernel=8, stage_cycles=(n if staged is not None else 0), **kw)
    assert L.shape()["kernel"] == 8
    if staged is not None:
        L.set_inputs(0, staged)
    else:
        L.set_seed(seed)
    hs, done = [], 0
    for k in list(chunks) + [n]:
        k = min(k, n - done)
        if k > 0:
            hs.append(L.step(k, hashes="host"))
            done += k
    H = np.concatenate(hs)
    F = L.read(list(range(c.n_signals)))
    r = oracle.simulate(c, n, seed=seed, lane0=kw.get("lane0", 0), n_lanes=nl, staged=staged, final=True)
    bad = np.argwhere(H != r.hashes)
    assert bad.shape[0] == 0, f"hash mismatch at (cycle, lane) {bad[:5].tolist()}"
    badf = np.argwhere(F != r.final_state)
    assert badf.shape[0] == 0, f"state mismatch at (signal, lane) {badf[:5].tolist()}"
    return L


@pytest.mark.gpu
@pytest.mark.parametrize("passes", [False, True])
def test_k8_c1_single_lane(rs, passes):
    cfg = CONFIGS["C1"]
    _check(rs, config_circuit("C1"), 300, 1, mode="single", passes=passes, seed=cfg.stim_seed, chunks=(1, 100))


@pytest.mark.gpu
@pytest.mark.parametrize("lt", [32, 64, 128])
def test_k8_c1_lanes(rs, lt):
    _check(rs, config_circuit("C1"), 40, 300, lane_tile=lt, lane0=17, seed=11, chunks=(7,))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1])
@pytest.mark.parametrize("mode", ["lanes", "single"])
def test_k8_edge_circuit_staged(rs, seed, mode):
    c = edge_circuit(seed)
    n, nl = 10, (150 if mode == "lanes" else 1)
    staged = edge_values(np.random.default_rng(300 + seed), (n, c.n_inputs, nl))
    _check(rs, c, n, nl, mode=mode, staged=staged, chunks=(3,))


@pytest.mark.gpu
def test_k8_fuzz_and_passes(rs):
    for seed in range(0, 40, 4):
        c = fuzz_circuit(seed)
        _check(rs, c, 25, 5, seed=seed, passes=bool(seed % 8), chunks=(2, 9))
    for seed in range(3):
        _check(rs, pass_circuit(seed), 12, 33, passes=True, seed=seed)


@pytest.mark.gpu
def test_k8_rejects_what_it_does_not_build(rs):
    g = rs.Graph(config_circuit("C1"), device=0, mode="single")
    with pytest.raises(rs.RtlSimError):
        rs.Lanes(g, 1, kernel=8, parts=2)
    L = rs.Lanes(g, 1, kernel=8)
    with pytest.raises(rs.RtlSimError, match="UNSUPPORTED|not built"):
        L.watch([0, 1])


@pytest.mark.gpu
@pytest.mark.parametrize("warps", [2, 3, 5, 8])
def test_k8_single_lane_multiwarp(rs, monkeypatch, warps):
    """Single lane split over several warps (shared-memory exchange, one named barrier per
    level): C1, the edge circuit with staged corner values, pass-rich and fuzz circuits."""
    monkeypatch.setenv("RTLSIM_K8_WARPS", str(warps))
    cfg = CONFIGS["C1"]
    L = _check(rs, config_circuit("C1"), 120, 1, mode="single", seed=cfg.stim_seed, chunks=(1, 50))
    assert L.shape()["threads"] == 32 * warps
    c = edge_circuit(warps % 2)
    staged = edge_values(np.random.default_rng(400 + warps), (9, c.n_inputs, 1))
    _check(rs, c, 9, 1, mode="single", staged=staged, chunks=(4,))
    _check(rs, pass_circuit(warps), 15, 1, mode="single", passes=True, seed=warps)
    for seed in range(warps, 40, 7):
        _check(rs, fuzz_circuit(seed), 20, 1, mode="single", seed=seed, chunks=(5,))
