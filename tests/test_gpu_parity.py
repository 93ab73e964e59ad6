"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Per-cycle, per-lane signal hashes (reading R12) plus full signal state via
rs_read_signals.  Integer work: the bar is bit equality everywhere.
"""
import json
import os

import numpy as np
import pytest

import oracle
from synth import CONFIGS, closed_form as cf, config_circuit, fuzz_circuit

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def run_gpu(rs, c, n_cycles, n_lanes=1, seed=0, mode="lanes", lane0=0, lane_tile=0, threads=0,
            staged=None, chunks=None, final=True, cluster=0, parts=0, kernel=0, repcut=0,
            repcut_global=False, l2_policy=0, op_pairs=0):
    g = rs.Graph(c, device=0, mode=mode)
    L = rs.Lanes(g, n_lanes, lane0=lane0, lane_tile=lane_tile, threads=threads, cluster=cluster,
                 stage_cycles=(n_cycles if staged is not None else 0), parts=parts, kernel=kernel,
                 repcut=repcut, repcut_global=repcut_global, l2_policy=l2_policy, op_pairs=op_pairs)
    if staged is not None:
        L.set_inputs(0, staged)
    else:
        L.set_seed(seed)
    hs = []
    for n in (chunks or [n_cycles]):
        hs.append(L.step(n, hashes="host"))
    H = np.concatenate(hs) if hs else np.zeros((0, n_lanes), np.uint64)
    F = L.read(list(range(c.n_signals))) if final else None
    return H, F, L


def check(rs, c, n_cycles, n_lanes=1, seed=0, mode="lanes", **kw):
    H, F, L = run_gpu(rs, c, n_cycles, n_lanes, seed, mode, **kw)
    lane0 = kw.get("lane0", 0)
    staged = kw.get("staged")
    r = oracle.simulate(c, n_cycles, seed=seed, lane0=lane0, n_lanes=n_lanes, staged=staged,
                        final=True, threads=8)
    if not np.array_equal(H, r.hashes):
        bad = np.argwhere(H != r.hashes)
        pytest.fail(f"hash mismatch at (cycle, lane) {bad[:5].tolist()} of {bad.shape[0]}")
    assert np.array_equal(F, r.final_state), np.argwhere(F != r.final_state)[:5]
    return L


def test_paper_example_both_modes(rs):
    c, outs = cf.paper_example(two_muls=True)
    for mode, kernel in (("lanes", 0), ("single", 0), ("single", 5)):
        H, F, _ = run_gpu(rs, c, 2, mode=mode, kernel=kernel)
        assert [int(F[o, 0]) for o in outs] == [4, 8]
        check(rs, c, 2, mode=mode, kernel=kernel)


def test_stimulus_matches_golden(rs):
    """The kernel's independent stimulus generator reproduces the golden values
    written by tests/golden/make_golden.py (oracle only)."""
    from synth import Builder
    b = Builder()
    ins = [b.input(64) for _ in range(4)]
    c = b.build()
    g = rs.Graph(c)
    L = rs.Lanes(g, 1024)
    L.set_seed(1)
    gold = json.load(open(os.path.join(HERE, "golden", "stimulus_seed1.json")))
    for cyc in range(3):
        L.step(1)
        vals = L.read(ins)
        for row in gold["values"]:
            if row["c"] == cyc:
                assert int(vals[row["k"], row["lane"]]) == int(row["value"]), row


@pytest.mark.parametrize("mode,kernel", [("lanes", 0), ("single", 0), ("single", 3), ("single", 4), ("single", 5)])
def test_c1_full(rs, mode, kernel):
    """C1 in every mode; single lane: auto (RepCut, one partition, since C1 fits
    one SM's shared memory), RepCut shared-memory / global, level-synchronous."""
    cfg = CONFIGS["C1"]
    L = check(rs, config_circuit("C1"), cfg.cycles, 1, seed=cfg.stim_seed, mode=mode, kernel=kernel)
    if mode == "single":
        assert L.shape()["kernel"] == (kernel or 3)


@pytest.mark.parametrize("kernel,lt,cs", [(2, 8, 1), (2, 16, 1), (2, 32, 1), (2, 32, 4), (2, 16, 2), (2, 8, 8),
                                          (1, 32, 1), (1, 64, 1), (1, 128, 1), (1, 32, 4), (1, 64, 2),
                                          (1, 128, 8), (6, 64, 1), (6, 128, 1), (6, 64, 2), (6, 128, 4),
                                          (6, 128, 8), (7, 32, 1), (7, 32, 4), (7, 64, 1), (7, 128, 1), (7, 64, 2),
                                          (7, 128, 4)])
def test_c2_structure_ragged_lanes(rs, lt, cs, kernel):
    """Full C2 circuit, 37 lanes (ragged last tile), 25 cycles, each lane tile,
    one CTA or a thread-block cluster per tile, both lane kernels."""
    check(rs, config_circuit("C2"), 25, 37, seed=CONFIGS["C2"].stim_seed, lane_tile=lt, cluster=cs,
          kernel=kernel)


@pytest.mark.parametrize("lt,cs,pairs", [(32, 1, 2), (32, 4, 2), (64, 2, 2), (128, 1, 2), (128, 4, 1), (64, 1, 1)])
def test_c2_kernel7_op_pairs(rs, lt, cs, pairs):
    """Kernel 7 with op pairs forced on (rs_lane_opts.op_pairs = 2; P = 1 included) or off."""
    check(rs, config_circuit("C2"), 25, 37, seed=CONFIGS["C2"].stim_seed, lane_tile=lt, cluster=cs, kernel=7,
          op_pairs=pairs)


@pytest.mark.parametrize("lt,pairs", [(128, 1), (64, 2), (32, 1)])
def test_c2_kernel7_cluster16(rs, lt, pairs):
    """Kernel 7 on 16-CTA (non-portable) clusters, ragged last tile."""
    check(rs, config_circuit("C2"), 25, 300, seed=CONFIGS["C2"].stim_seed, lane_tile=lt, cluster=16, kernel=7,
          op_pairs=pairs)


def test_c2_threads_variants(rs):
    c = config_circuit("C2", n_ops=5000, n_levels=40, n_regs=500)
    for th in (64, 256, 512):
        check(rs, c, 12, 40, seed=7, threads=th, lane_tile=8, kernel=2)
    for th in (32, 96, 640):
        check(rs, c, 12, 70, seed=7, threads=th, lane_tile=64, kernel=1)
    for th in (32, 160, 768):
        check(rs, c, 12, 200, seed=7, threads=th, lane_tile=128, kernel=6)
        check(rs, c, 12, 200, seed=7, threads=th, lane_tile=128, kernel=7)


@pytest.mark.parametrize("kernel", [1, 2, 6, 7])
def test_c3_structure(rs, kernel):
    check(rs, config_circuit("C3"), 6, 40, seed=CONFIGS["C3"].stim_seed, kernel=kernel)


def test_c5_structure_single_lane(rs):
    """C5 generator, scaled to 200k ops / 150 levels, single-lane grid mode."""
    c = config_circuit("C5", n_ops=200_000, n_regs=25_000, n_inputs=512)
    check(rs, c, 12, 1, seed=CONFIGS["C5"].stim_seed, mode="single")


def test_fuzz_corpus(rs):
    """Fuzz corpus (SPEC.md S:405 shape): constants, register->source edges,
    wide folds, permuted ids; 60 cycles, both modes."""
    for seed in range(200):
        c = fuzz_circuit(seed)
        check(rs, c, 60, 3, seed=seed, kernel=(1, 2, 6, 7)[seed % 4])
        if seed % 4 == 0:
            check(rs, c, 60, 1, seed=seed, mode="single", kernel=5 if seed % 8 else 0)


def test_closed_forms_on_gpu(rs):
    c, r = cf.counter(13)
    H, F, _ = run_gpu(rs, c, 300, 4)
    assert (F[r] == 300 % 2 ** 13).all()
    c, s = cf.lfsr(16, (16, 14, 13, 11), seed=1)
    H, F, L = run_gpu(rs, c, 65535, 2)
    assert (F[s] == 1).all()                             # period 2^16 - 1
    r0 = oracle.simulate(c, 65535, n_lanes=1)
    for kernel in (0, 5):
        H1, F1, _ = run_gpu(rs, c, 65535, 1, mode="single", final=True, kernel=kernel)
        assert int(F1[s, 0]) == 1
        assert np.array_equal(H1, r0.hashes) and np.array_equal(H[:, :1], r0.hashes)
    c, a, b, out = cf.ripple_adder(8)
    A = np.repeat(np.arange(256, dtype=np.uint64), 256)
    B = np.tile(np.arange(256, dtype=np.uint64), 256)
    H, F, _ = run_gpu(rs, c, 1, 65536, staged=np.stack([A, B])[None])
    assert np.array_equal(F[out], A + B)
    c, x, regs = cf.shift_register(6, 16)
    vals = (np.arange(40, dtype=np.uint64) * np.uint64(977) + np.uint64(5))[:, None, None]
    check(rs, c, 40, 1, staged=vals)


@pytest.mark.parametrize("kernel", [1, 2, 6, 7])
def test_chunking_and_hash_toggle(rs, kernel):
    c = config_circuit("C2", n_ops=4000, n_levels=20, n_regs=400)
    g = rs.Graph(c)
    L = rs.Lanes(g, 50, kernel=kernel)
    L.set_seed(11)
    h1 = L.step(7, hashes="host")
    L.step(5)                                             # hash off: carry must be refreshed
    h3 = L.step(8, hashes="host")
    h4 = L.step(1, hashes="host")
    r = oracle.simulate(c, 21, seed=11, n_lanes=50)
    assert np.array_equal(h1, r.hashes[:7])
    assert np.array_equal(h3, r.hashes[12:20]) and np.array_equal(h4, r.hashes[20:21])
    assert L.cycle == 21
    L.step(0)
    assert L.cycle == 21


@pytest.mark.parametrize("kernel", [1, 6, 7])
@pytest.mark.parametrize("cluster", [1, 2])
def test_wide_work_items(rs, cluster, kernel):
    """Kernels 1 and 6 with kBatchWide-op work items (>= 2,048 ops per CTA and
    level: cluster 1) and with kBatch-op items (cluster 2), ragged lanes."""
    c = config_circuit("C3", n_ops=60000, n_levels=20, n_regs=3000)
    check(rs, c, 5, 70, seed=9, kernel=kernel, lane_tile=64, cluster=cluster)


@pytest.mark.parametrize("mode,kernel", [("lanes", 1), ("lanes", 2), ("lanes", 6), ("lanes", 7), ("single", 0),
                                         ("single", 5)])
def test_staged_inputs_pipelined(rs, mode, kernel):
    """The next chunk is staged (copy stream) before the current one is stepped,
    with a ring of two chunks: every copy must wait for the launch that last
    read its slots, every step for the copies before it."""
    c = config_circuit("C2", n_ops=3000, n_levels=15, n_regs=300) if mode == "lanes" else config_circuit("C1")
    rng = np.random.default_rng(5)
    n, ch = 60, 6
    nl = (33 if kernel == 2 else 130) if mode == "lanes" else 1
    vals = rng.integers(0, 2**63, size=(n, c.n_inputs, nl), dtype=np.int64).astype(np.uint64)
    g = rs.Graph(c, mode=mode)
    L = rs.Lanes(g, nl, stage_cycles=2 * ch, kernel=kernel)
    L.set_inputs(0, vals[0:ch])
    hs = []
    for c0 in range(0, n, ch):
        if c0 + ch < n:
            L.set_inputs(c0 + ch, vals[c0 + ch:c0 + 2 * ch])
        hs.append(L.step(ch, hashes="host"))
    r = oracle.simulate(c, n, n_lanes=nl, staged=vals)
    assert np.array_equal(np.concatenate(hs), r.hashes)
    F = L.read(list(range(c.n_signals)))
    assert np.array_equal(F, oracle.simulate(c, n, n_lanes=nl, staged=vals, final=True).final_state)


def test_staged_inputs_from_device_stream(rs):
    """Device-resident stimulus produced by kernels on the lanes' stream and
    staged right away (no host sync): the copy must follow that work."""
    import torch
    c = config_circuit("C2", n_ops=2000, n_levels=10, n_regs=200)
    n, nl = 24, 96
    vals = np.random.default_rng(2).integers(0, 2**62, size=(n, c.n_inputs, nl), dtype=np.int64)
    st = torch.cuda.Stream()
    g = rs.Graph(c)
    L = rs.Lanes(g, nl, stage_cycles=n, stream=st, kernel=2)
    with torch.cuda.stream(st):
        base = torch.from_numpy(vals).cuda()
        for _ in range(8):                 # a queue of kernels producing the values
            base = base * 3 - base * 2
        t = base.view(torch.uint64) if hasattr(torch, "uint64") else base
        L.set_inputs(0, t)
        H = L.step(n, hashes="host")
    r = oracle.simulate(c, n, n_lanes=nl, staged=vals.astype(np.uint64))
    assert np.array_equal(H, r.hashes)


@pytest.mark.parametrize("kernel", [1, 2, 6, 7])
def test_staged_inputs_chunks(rs, kernel):
    c = config_circuit("C2", n_ops=3000, n_levels=15, n_regs=300)
    rng = np.random.default_rng(3)
    n, nl = 30, 33 if kernel == 2 else 130
    vals = rng.integers(0, 2**63, size=(n, c.n_inputs, nl), dtype=np.int64).astype(np.uint64) * np.uint64(3)
    g = rs.Graph(c)
    L = rs.Lanes(g, nl, stage_cycles=8, kernel=kernel)
    hs = []
    for c0 in range(0, n, 6):
        L.set_inputs(c0, vals[c0:c0 + 6])
        hs.append(L.step(6, hashes="host"))
    r = oracle.simulate(c, n, n_lanes=nl, staged=vals)
    assert np.array_equal(np.concatenate(hs), r.hashes)
    with pytest.raises(rs.RtlSimError) as e:
        L.step(3)                                         # cycles 30..32 not staged
    assert e.value.name == "RS_E_STATE"


@pytest.mark.parametrize("kernel", [1, 2, 6, 7])
def test_checkpoint_restore(rs, kernel):
    c = config_circuit("C2", n_ops=3000, n_levels=15, n_regs=300)
    full = oracle.simulate(c, 20, seed=5, n_lanes=24)
    g = rs.Graph(c)
    a = rs.Lanes(g, 24, kernel=kernel)
    a.set_seed(5)
    h0 = a.step(10, hashes="host")
    regs = a.read(c.reg_id)
    b = rs.Lanes(g, 24, kernel={1: 2, 2: 6, 6: 7, 7: 1}[kernel])   # restored into another lane kernel's layout
    b.set_seed(5)
    b.write_registers(c.reg_id, regs)
    b.cycle = 10
    h1 = b.step(10, hashes="host")
    assert np.array_equal(np.concatenate([h0, h1]), full.hashes)
    with pytest.raises(rs.RtlSimError) as e:
        b.write_registers([int(c.input_id[0])], np.zeros((1, 24), np.uint64))
    assert e.value.name == "RS_E_RANGE"


def test_lane_sharding_invariance(rs):
    """Global lane ids: two shards (lane0 = 0, 37) reproduce one 74-lane run
    (the multi-GPU partition of SURVEY §8(e))."""
    c = config_circuit("C2", n_ops=3000, n_levels=15, n_regs=300)
    Hf, Ff, _ = run_gpu(rs, c, 15, 74, seed=9)
    Ha, Fa, _ = run_gpu(rs, c, 15, 37, seed=9, lane0=0)
    Hb, Fb, _ = run_gpu(rs, c, 15, 37, seed=9, lane0=37)
    assert np.array_equal(Hf, np.concatenate([Ha, Hb], axis=1))
    assert np.array_equal(Ff, np.concatenate([Fa, Fb], axis=1))
    # the same partition across the two lane kernels (shards may run different layouts)
    Hc, Fc, _ = run_gpu(rs, c, 15, 37, seed=9, lane0=37, kernel=1)
    assert np.array_equal(Hb, Hc) and np.array_equal(Fb, Fc)
    Hd, Fd, _ = run_gpu(rs, c, 15, 37, seed=9, lane0=37, kernel=6)
    assert np.array_equal(Hb, Hd) and np.array_equal(Fb, Fd)
    He, Fe, _ = run_gpu(rs, c, 15, 37, seed=9, lane0=37, kernel=7)
    assert np.array_equal(Hb, He) and np.array_equal(Fb, Fe)


def test_error_statuses(rs):
    c = config_circuit("C1")
    g = rs.Graph(c)
    L = rs.Lanes(g, 4)
    with pytest.raises(rs.RtlSimError) as e:
        L.read([0], lane_begin=3, n_lanes=2)
    assert e.value.name == "RS_E_RANGE"
    with pytest.raises(rs.RtlSimError) as e:
        L.read([c.n_signals])
    assert e.value.name == "RS_E_RANGE"
    with pytest.raises(rs.RtlSimError) as e:
        L.set_inputs(0, np.zeros((1, c.n_inputs, 4), np.uint64))
    assert e.value.name == "RS_E_STATE"
    gs = rs.Graph(c, mode="single")
    with pytest.raises(rs.RtlSimError) as e:
        rs.Lanes(gs, 2)
    assert e.value.name == "RS_E_INVALID_ARG"
    with pytest.raises(rs.RtlSimError) as e:
        rs.Lanes(g, 0)
    assert e.value.name == "RS_E_INVALID_ARG"


def test_degenerate_graphs(rs):
    from synth import Builder
    b = Builder()                                   # registers only, no ops
    r = b.reg(8, 3)
    b.set_next(r, r)
    check(rs, b.build(), 5, 3)
    b = Builder()                                   # inputs only
    b.input(12)
    b.input(64)
    check(rs, b.build(), 5, 70, seed=4)
    b = Builder()                                   # constants feeding ops, no inputs
    k = b.const(64, 2**64 - 1)
    k2 = b.const(7, 5)
    b.op("add", [k, k2], 64)
    b.op("cat", [k2, k], 64)
    c = b.build()
    for mode, kernel in (("lanes", 0), ("single", 0), ("single", 5)):
        check(rs, c, 3, 1, mode=mode, kernel=kernel)


@pytest.mark.slow
def test_full_size_sampled(rs):
    """BASELINE.json full sizes in the bench's launch configuration (auto
    lane tile / threads): GPU runs all lanes; the oracle checks sampled
    lanes (first/last of tiles, spread) cycle by cycle."""
    for name, cycles, sample in (("C2", 60, 12), ("C3", 6, 6)):
        cfg = CONFIGS[name]
        c = config_circuit(name)
        H, _, L = run_gpu(rs, c, cycles, cfg.lanes, seed=cfg.stim_seed, final=False)
        lt = L.shape()["lane_tile"]
        lanes = sorted(set([0, lt - 1, lt, cfg.lanes - 1] +
                           list(np.linspace(0, cfg.lanes - 1, sample).astype(int))))
        r = oracle.simulate(c, cycles, seed=cfg.stim_seed, lanes=lanes, threads=8)
        assert np.array_equal(H[:, lanes], r.hashes), name
        F = L.read(list(range(0, c.n_signals, 7)))
        rf = oracle.simulate(c, cycles, seed=cfg.stim_seed, lanes=lanes[:3], final=True, hashes=False)
        assert np.array_equal(F[:, lanes[:3]], rf.final_state[::7])


@pytest.mark.slow
def test_c4_c5_full_size_sampled(rs):
    c = config_circuit("C4")
    cfg = CONFIGS["C4"]
    H, _, L = run_gpu(rs, c, 2, cfg.lanes, seed=cfg.stim_seed, final=False)
    lanes = [0, 31, 4096, cfg.lanes - 1]
    r = oracle.simulate(c, 2, seed=cfg.stim_seed, lanes=lanes, threads=4)
    assert np.array_equal(H[:, lanes], r.hashes)
    del L
    c = config_circuit("C5")
    H, F, _ = run_gpu(rs, c, 10, 1, seed=CONFIGS["C5"].stim_seed, mode="single", final=True)
    r = oracle.simulate(c, 10, seed=CONFIGS["C5"].stim_seed, final=True)
    assert np.array_equal(H, r.hashes) and np.array_equal(F, r.final_state)


def test_auto_kernel_choice(rs):
    """rs_lane_opts.kernel = 0: kernel 7 (records, 32 * P-lane tiles) at >= 2048 lanes; below,
    kernel 2 -- except for designs with <= 1,024 ops per level at >= 1,024 or <= 256 lanes,
    which take kernel 7's 32-lane tiles (runtime.cu, profiles/r02/k7low)."""
    c = config_circuit("C2", n_ops=2000, n_levels=10, n_regs=100)      # 200 ops per level
    cw = config_circuit("C2", n_ops=12000, n_levels=8, n_regs=100)     # 1,500 ops per level
    g, gw = rs.Graph(c), rs.Graph(cw)
    a = rs.Lanes(gw, 1024)
    b = rs.Lanes(g, 4096)
    d = rs.Lanes(g, 1024)
    e = rs.Lanes(g, 512)
    f = rs.Lanes(g, 200)
    assert a.shape()["kernel"] == 2 and a.shape()["lane_tile"] in (8, 16, 32)
    assert b.shape()["kernel"] == 7 and b.shape()["lane_tile"] in (64, 128)
    assert d.shape()["kernel"] == 7 and d.shape()["lane_tile"] == 32
    assert e.shape()["kernel"] == 2
    assert f.shape()["kernel"] == 7 and f.shape()["lane_tile"] == 32
    for L, cc in ((a, cw), (b, c), (d, c), (e, c), (f, c)):
        L.set_seed(3)
        h = L.step(3, hashes="host")
        r = oracle.simulate(cc, 3, seed=3, lanes=[0, L.n_lanes - 1], threads=2)
        assert np.array_equal(h[:, [0, L.n_lanes - 1]], r.hashes)


@pytest.mark.parametrize("kernel", [1, 2, 6, 7])
def test_waveform_changes(rs, kernel):
    """Waveform capture (rs_watch): the fused per-cycle change
    records equal the change set of the oracle's per-cycle trace of the same
    signals (ops, inputs, registers of every width class), across step chunks
    and a re-armed watch."""
    from paper_2601_18140_b200.wave import changes_from_trace
    c = config_circuit("C2", n_ops=3000, n_levels=15, n_regs=300)
    rng = np.random.default_rng(kernel)
    ids = sorted(set(rng.choice(c.n_signals, 40, replace=False).tolist()) | {int(c.input_id[0]), int(c.reg_id[0])})
    nl = 45 if kernel == 2 else 140
    g = rs.Graph(c)
    L = rs.Lanes(g, nl, lane0=1000, kernel=kernel)
    L.set_seed(4)
    L.step(3)                                  # not watched
    L.watch(ids, capacity=1 << 20)
    L.step(5)
    L.step(7, hashes="host")
    rec, dropped = L.wave_read()
    assert dropped == 0
    got = {(int(r["cycle"]), int(r["lane"]), int(r["watch"]), int(r["value"])) for r in rec}
    assert len(got) == len(rec)
    lanes = list(range(1000, 1000 + nl))
    tr = oracle.simulate(c, 15, seed=4, lane0=1000, n_lanes=nl, watch=ids, hashes=False).trace
    assert got == changes_from_trace(tr[3:], 3, lanes)
    # re-arm on a subset: records restart from the current cycle
    L.watch(ids[:5], capacity=64)
    L.step(4)
    rec, dropped = L.wave_read()
    exp = changes_from_trace(
        oracle.simulate(c, 19, seed=4, lane0=1000, n_lanes=nl, watch=ids[:5], hashes=False).trace[15:], 15, lanes)
    assert len(rec) == 64 and dropped == len(exp) - 64
    got = {(int(r["cycle"]), int(r["lane"]), int(r["watch"]), int(r["value"])) for r in rec}
    assert got <= exp
    L.watch([])
    L.step(2)
    assert L.wave_read()[0].shape[0] == 0


@pytest.mark.parametrize("kw", [dict(kernel=5), dict(), dict(repcut=3), dict(kernel=5, name="C5s")])
def test_waveform_single_lane(rs, kw):
    """Single-lane waveform capture: the level-synchronous grid and RepCut
    (shared-memory slices; watched signals read by the partition that holds
    them) record exactly the oracle trace's changes."""
    from paper_2601_18140_b200.wave import changes_from_trace
    kw = dict(kw)
    name = kw.pop("name", "C1")
    c = config_circuit("C1") if name == "C1" else config_circuit("C5", n_ops=20000, n_levels=30, n_regs=2000)
    rng = np.random.default_rng(3)
    ids = sorted(set(rng.choice(c.n_signals, 30, replace=False).tolist()) | {int(c.input_id[0]), int(c.reg_id[0])})
    g = rs.Graph(c, mode="single")
    L = rs.Lanes(g, 1, **kw)
    L.set_seed(6)
    L.step(2)
    L.watch(ids, capacity=1 << 16)
    L.step(4)
    L.step(9, hashes="host")
    rec, dropped = L.wave_read()
    assert dropped == 0
    got = {(int(r["cycle"]), int(r["lane"]), int(r["watch"]), int(r["value"])) for r in rec}
    assert len(got) == len(rec)
    tr = oracle.simulate(c, 15, seed=6, n_lanes=1, watch=ids, hashes=False).trace
    assert got == changes_from_trace(tr[2:], 2, [0])
    H = oracle.simulate(c, 15, seed=6, n_lanes=1).hashes
    L2 = rs.Lanes(g, 1, **kw)
    L2.set_seed(6)
    assert np.array_equal(L2.step(15, hashes="host"), H)


def test_watch_errors(rs):
    c = config_circuit("C1")
    g = rs.Graph(c)
    L = rs.Lanes(g, 4)
    with pytest.raises(rs.RtlSimError) as e:
        L.watch([c.n_signals])
    assert e.value.name == "RS_E_RANGE"
    with pytest.raises(rs.RtlSimError) as e:
        L.watch([0], capacity=0)
    assert e.value.name == "RS_E_INVALID_ARG"
    gs = rs.Graph(c, mode="single")
    for kw in (dict(parts=2), dict(repcut=2, repcut_global=True)):
        Ls = rs.Lanes(gs, 1, **kw)
        with pytest.raises(rs.RtlSimError) as e:
            Ls.watch([0])
        assert e.value.name == "RS_E_UNSUPPORTED"
    assert L.wave_read()[0].shape[0] == 0           # nothing watched: empty


@pytest.mark.parametrize("policy", [1, 2])
@pytest.mark.parametrize("kernel", [1, 2, 6, 7])
def test_l2_policy_results_identical(rs, policy, kernel):
    """rs_lane_opts.l2_policy (access-policy window over the schedule / the state) changes
    speed only."""
    c = config_circuit("C3", n_ops=20000, n_levels=20, n_regs=2000)
    check(rs, c, 8, 150, seed=4, kernel=kernel, l2_policy=policy)


@pytest.mark.parametrize("kernel", [1, 2, 6, 7])
def test_caller_owned_state(rs, kernel):
    """rs_lane_opts.defer_state + rs_lanes_bind_state (SURVEY.md §8(b) torch-owned memory):
    the signal state lives in a torch tensor; results equal the oracle's, and the library
    refuses to step before the state is bound or with a too-small buffer."""
    import torch
    c = config_circuit("C2", n_ops=3000, n_levels=15, n_regs=300)
    g = rs.Graph(c)
    L = rs.Lanes(g, 50, kernel=kernel, state="torch")
    assert L.state.is_cuda and L.state.numel() == L.state_bytes()
    L.set_seed(8)
    h = L.step(9, hashes="host")
    r = oracle.simulate(c, 9, seed=8, n_lanes=50, final=True)
    assert np.array_equal(h, r.hashes)
    assert np.array_equal(L.read(list(range(c.n_signals))), r.final_state)
    M = rs.Lanes(g, 50, kernel=kernel)          # library-owned state: same size
    assert M.state_bytes() == L.state_bytes()
    import ctypes
    opts = rs.LaneOpts(0, 0, 0, 0, 0, None, 0, kernel, 0, 0, 0, 0, 0, 1)
    hnd = ctypes.c_void_p()
    rs._check(rs.lib().rs_alloc_lanes(g.h, 50, ctypes.byref(opts), ctypes.byref(hnd)))
    with pytest.raises(rs.RtlSimError) as e:
        rs._check(rs.lib().rs_step_cycles(hnd, 1, None, 0))
    assert e.value.name == "RS_E_STATE"
    small = torch.empty(256, dtype=torch.uint8, device="cuda")
    with pytest.raises(rs.RtlSimError) as e:
        rs._check(rs.lib().rs_lanes_bind_state(hnd, ctypes.c_void_p(small.data_ptr()), 256))
    assert e.value.name == "RS_E_CAPACITY"
    rs.lib().rs_free_lanes(hnd)
