#!/usr/bin/env python
"""Benchmark: simulated lane-cycles/s of the B200 RTeAAL Sim hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference]

One step = one rs_step_cycles launch over the config's full cycle count for
this rank's lanes (inject -> every level's gather/op/write -> hash -> commit,
all cycles), hashes on.  Default workload: C3, the largest BASELINE.json
config that fits one GPU (4,096 lanes x 10,000 cycles).

N > 1: one process per GPU.  Under torchrun the ranks come from the
environment; a plain `python bench.py --gpus N` re-executes itself under
torch.distributed.run.  Lane configs are split into contiguous global lane
ranges [d*L/N, (d+1)*L/N) (`--scaling strong`, the default)
or give every rank the config's lane count (`--scaling weak`).  There is no
data-path collective: lanes are independent; a gloo process group carries the
barriers around the timed region and the max-over-ranks reduction only (so it
also works with several ranks on one device).  Single-lane configs (C1, C5,
MC16) run one independent replica per rank at N > 1.

Timing: CUDA events on the launching stream around each step, barrier +
synchronize on both sides of the timed region, max over ranks; L2 flushed
(256 MB write) before every timed step.  `value` = all ranks' lane-cycles /
the max-over-ranks device time of the K steps; `ms_per_step_median` is the
median step.  A hash-off pass (pure throughput) follows.
`--impl reference` times the CPU oracle (test infrastructure, oracle/) on
the host cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated lane-cycles/s and op-evals/s at 1/2/4/8 B200; % of BW roofline"
UNIT = "lane-cycles/s"
SINGLE = ("C1", "C5", "MC16")
# per-config roofline bound (SURVEY.md §8(d) "Roofline quantities"): HBM when the
# per-GPU state exceeds L2 (C3, C4); L2 when state + graph fit (C2); single-lane
# configs are latency-bound (reported against HBM, with the latency floor in DESIGN.md)
BOUND = {"C1": "hbm", "C2": "l2", "C3": "hbm", "C4": "hbm", "C5": "hbm", "MC16": "hbm"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_l2_peak():
    """Measured L2 read bandwidth at a 64 MiB working set (tools/microbench.cu on a
    B200, stored in profiles/)."""
    for rnd in ("r02", "r01"):
        p = os.path.join(ROOT, "profiles", rnd, "microbench.json")
        if os.path.exists(p):
            d = json.load(open(p))
            return float(d["read_bw_gbs"]["64_MiB"]), f"measured L2 read BW at 64 MiB (profiles/{rnd}/microbench.json)"
    return None, "unmeasured"


def load_traffic(cfg_name, lanes, cycles, kernel):
    """DRAM bytes of the dominant kernel per launch, scaled from the stored ncu --set
    full capture of the same kernel (profiles/<round>/traffic_<cfg>.json); tagged as stored."""
    for rnd in ("r02", "r01", ""):
        p = os.path.join(ROOT, "profiles", rnd, f"traffic_{cfg_name}.json")
        if os.path.exists(p):
            t = json.load(open(p))
            per = t.get("dram_bytes_per_lane_cycle")
            if not per:
                return None, None
            src = (f"stored: {os.path.relpath(p, ROOT)} (ncu --set full, kernel {t.get('kernel')}, "
                   f"{t.get('lanes')} lanes x {t.get('cycles')} cycles), scaled to this launch")
            return per * lanes * cycles, src
    return None, None


class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def workload(cfg_name, total_lanes, lanes_rank, cycles, n_ops, n_levels, n_gpus, scaling, levelcut=False):
    if cfg_name in SINGLE:
        how = (f", level cut across {n_gpus} GPUs" if levelcut else f", {n_gpus} independent replicas") \
            if n_gpus > 1 else ""
        return (f"{cfg_name}: {n_ops} ops / {n_levels} levels, 1 lane x {cycles} cycles per step"
                + how + ", synthetic seeded circuit + stimulus")
    return (f"{cfg_name}: {n_ops} ops / {n_levels} levels, {total_lanes} lanes x {cycles} cycles per step, "
            f"{n_gpus} GPU(s) ({lanes_rank} lanes per GPU, {scaling} scaling), synthetic seeded circuit + stimulus")


def oracle_rate(circ, seed, n_lanes, n_cycles, lane0=0, threads=1):
    import oracle
    t = time.perf_counter()
    oracle.simulate(circ, n_cycles, seed=seed, lane0=lane0, n_lanes=n_lanes, threads=threads)
    dt = time.perf_counter() - t
    return n_lanes * n_cycles / dt, dt


def cpu_sample_plan(circ, target_s, cores):
    """Lanes x cycles of oracle work taking about target_s on `cores` threads
    (calibrated with a short run)."""
    import oracle
    lanes = max(1, cores)
    n = 2
    while True:  # calibrate on at least ~0.2 s of work (tiny circuits run thousands of cycles per ms)
        t = time.perf_counter()
        oracle.simulate(circ, n, seed=1, n_lanes=lanes, threads=cores)
        dt = time.perf_counter() - t
        if dt > 0.2 or n >= 1 << 20:
            break
        n *= 8
    per_cycle = max(dt / n, 1e-9)
    cycles = int(max(2, min(10_000_000, target_s / per_cycle)))
    return lanes, cycles


def get_config(name):
    from synth import CONFIGS, config_circuit, multicore_circuit
    if name == "MC16":
        import types
        circ = multicore_circuit()
        cfg = types.SimpleNamespace(name="MC16", lanes=1, cycles=2000, stim_seed=circ.meta["stim_seed"], n_levels=60)
    else:
        cfg = CONFIGS[name]
        circ = config_circuit(name)
    return cfg, circ


def run_reference(args, cfg, circ):
    """--impl reference: the oracle (as it stands) on the host cores; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    lanes, cycles = cpu_sample_plan(circ, args.ref_step_s, cores)
    for w in range(args.warmup):
        oracle_rate(circ, cfg.stim_seed, lanes, max(2, cycles // 10), threads=cores)
    tot = 0.0
    for k in range(args.steps):
        _, dt = oracle_rate(circ, cfg.stim_seed, lanes, cycles, lane0=k * lanes, threads=cores)
        tot += dt
    value = lanes * cycles * args.steps / tot
    total_lanes = 1 if args.config in SINGLE else (args.lanes or cfg.lanes)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.config in SINGLE else args.scaling,
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": workload(cfg.name, total_lanes, total_lanes, args.cycles or cfg.cycles, circ.n_ops,
                                        cfg.n_levels, args.gpus, args.scaling)},
        "op_evals_per_s": value * circ.n_ops,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{lanes} lanes x {cycles} cycles per step (one lane per thread)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(n):
    """Re-execute this command under torch.distributed.run with n ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def time_steps(L, stream, cycles, hashes, steps, flush, barrier, torch):
    evs = []
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    l0 = L.launches
    for _ in range(steps):
        flush.fill_(1)                          # L2 flush between timed steps
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        L.step(cycles, hashes=hashes)
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs], L.launches - l0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5", "MC16"],
                    help="BASELINE configs; MC16 = synth.multicore_circuit() (16 cores x 12.5k ops, the RepCut "
                         "workload of SURVEY.md §8(f) NEXT-2)")
    ap.add_argument("--cycles", type=int, default=0, help="cycles per step (default: the config's)")
    ap.add_argument("--lanes", type=int, default=0, help="total lanes (strong) / lanes per GPU (weak); "
                                                         "default: the config's")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-hash", action="store_true", help="time the hash-off step as the headline")
    ap.add_argument("--no-passes", action="store_true",
                    help="compile without the constant / copy propagation passes (RS_LOAD_PASSES)")
    ap.add_argument("--no-hash-off-pass", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--lane-tile", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--cluster", type=int, default=0)
    ap.add_argument("--kernel", type=int, default=0, help="rs_lane_opts.kernel (0 auto; C1 defaults to 8, specialised)")
    ap.add_argument("--parts", type=int, default=0, help="C1/C5: level-cut partitions emulated on this GPU")
    ap.add_argument("--repcut", type=int, default=0, help="single-lane configs: RepCut partitions (rs_lane_opts.repcut)")
    ap.add_argument("--repcut-global", type=int, default=0,
                    help="rs_lane_opts.repcut_global (0 auto, 1 the global-memory RepCut kernel, 2 shared-memory slices)")
    ap.add_argument("--ref-step-s", type=float, default=4.0)
    ap.add_argument("--watch", type=int, default=0, help="waveform capture of N signals during the timed steps")
    ap.add_argument("--op-pairs", type=int, default=0, help="rs_lane_opts.op_pairs (kernel 7: 0 auto, 1 off, 2 on)")
    ap.add_argument("--l2-policy", type=int, default=0, help="rs_lane_opts.l2_policy (0 none, 1 schedule, 2 state)")
    ap.add_argument("--replicas", action="store_true",
                    help="C1/C5 at N > 1: independent replicas instead of the level cut across GPUs")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)

    cfg, circ = get_config(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg, circ)

    import torch
    import torch.distributed as tdist
    from paper_2601_18140_b200 import dist as D
    from paper_2601_18140_b200 import rtlsim as rs

    rank, world, local = D.env_rank()
    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev                    # more ranks than GPUs: ranks share devices (independent lanes)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        tdist.init_process_group("gloo")  # barriers + timing reduction only; no data-path collective
        dist = tdist

    single = args.config in SINGLE
    cycles = args.cycles or cfg.cycles
    if single:
        shard = D.Shard(rank, world, 0, 1)
        total_lanes = 1
    elif args.scaling == "strong":
        total_lanes = args.lanes or cfg.lanes
        shard = D.shard_strong(rank, world, total_lanes)
    else:
        shard = D.shard_weak(rank, world, args.lanes or cfg.lanes)
        total_lanes = shard.n_lanes * world
    lanes = shard.n_lanes
    # C1 / C5 at N > 1: the level cut across the ranks' GPUs, one
    # partition per rank, peer-mapped replicas and flags (rs_ipc_connect); ranks sharing a
    # device would wait on one another, so that case falls back to independent replicas
    levelcut = single and world > 1 and args.config in ("C1", "C5") and not args.replicas and ndev >= world
    stream = torch.cuda.Stream()
    g = rs.Graph(circ, device=dev, mode="single" if single else "lanes", passes=not args.no_passes)
    info = g.info()
    info0 = rs.Graph(circ, device=rs.RS_DEVICE_NONE, mode="single" if single else "lanes").info()
    kernel = args.kernel
    if kernel == 0 and args.config == "C1" and args.parts <= 1 and not args.repcut and not args.watch:
        kernel = 8  # C1 fits the specialised kernel (rs_specialize): 1.02 vs 4.07 us per cycle (RepCut)
    mk = dict(lane0=shard.lane0, lane_tile=args.lane_tile, threads=args.threads, stream=stream,
              cluster=args.cluster, parts=args.parts, kernel=kernel, repcut=args.repcut,
              **({"repcut_global": args.repcut_global} if args.repcut_global else {}),
              l2_policy=args.l2_policy if not single else 0, op_pairs=args.op_pairs)
    if levelcut:
        L = rs.Lanes(g, 1, stream=stream, part_world=world, part_rank=rank)
        hs = [None] * world
        dist.all_gather_object(hs, L.ipc_handle())
        L.ipc_connect(hs)
        dist.barrier()
    else:
        L = rs.Lanes(g, lanes, **mk)
    L.set_seed(cfg.stim_seed)
    if args.watch:
        wids = np.linspace(0, circ.n_signals - 1, args.watch).astype(np.uint32)
        L.watch(wids, capacity=1 << 26)
    hbuf = torch.empty(cycles * lanes, dtype=torch.int64, device="cuda")
    hashes = None if args.no_hash else hbuf
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")

    def barrier():
        if dist is not None:
            dist.barrier()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            L.step(cycles, hashes=hashes)
        with ClockSampler(dev) as clk:
            step_ms, launches = time_steps(L, stream, cycles, hashes, args.steps, flush, barrier, torch)
        hash_off = None
        if not args.no_hash and not args.no_hash_off_pass:
            n_off = max(1, min(args.steps, 3))
            L.step(cycles)                                   # warm the hash-off variant
            off_ms, _ = time_steps(L, stream, cycles, None, n_off, flush, barrier, torch)
            hash_off = off_ms
    total_ms = D.max_over_ranks(float(sum(step_ms)), dist)
    med_ms = D.max_over_ranks(float(np.median(step_ms)), dist)
    n_replicas = world if (single and not levelcut) else 1
    all_lane_cycles = (total_lanes * n_replicas if single else total_lanes) * cycles * args.steps
    value = all_lane_cycles / (total_ms / 1e3)

    kid = L.shape()["kernel"]
    kernel_name = {1: "k_lanes_t", 2: "k_lanes", 3: "k_repcut_smem", 4: "k_repcut", 5: "k_single2", 6: "k_lanes_b",
                   7: "k_lanes_r", 8: "rs_su (specialised PTX)"}.get(kid, "?")
    # roofline of the dominant (only) kernel: algorithmic bytes per launch / launch duration
    # (this rank's launch; the max-over-ranks time)
    bytes_per_cycle = lanes * info["alg_bytes_per_lane_cycle"] + info["graph_alg_bytes"]
    alg_bytes = bytes_per_cycle * cycles
    kern_s = (total_ms / args.steps) / 1e3
    bound = BOUND[args.config]
    if bound == "l2":
        peak, peak_src = load_l2_peak()
        if peak is None:
            bound = "hbm"
    if bound == "hbm":
        peak, peak_src = load_peaks()
    achieved = alg_bytes / kern_s / 1e9
    traffic, traffic_src = load_traffic(args.config, lanes, cycles, kid)

    # end to end through the public API with host buffers: staged inputs H2D from
    # pinned memory and hashes D2H, every chunk, inside the timed region.
    e2e = None
    if not args.no_e2e and not levelcut:
        chunk = min(cycles, max(1, (256 << 20) // max(1, 8 * circ.n_inputs * lanes)))
        Ls = rs.Lanes(g, lanes, stage_cycles=2 * chunk, **mk)
        rng = np.random.default_rng(rank)
        host_in = torch.from_numpy(rng.integers(0, 2**63, size=(chunk, circ.n_inputs, lanes),
                                                dtype=np.int64)).pin_memory()
        host_h = torch.empty((chunk, lanes), dtype=torch.int64).pin_memory()
        in_np = host_in.numpy().view(np.uint64)
        h_np = host_h.numpy().view(np.uint64)

        def e2e_step():
            # double-buffered ring: chunk k+1's inputs are copied (the library's copy
            # stream) while chunk k is simulated; hashes come back per chunk
            c0, done, staged = Ls.cycle, 0, min(chunk, cycles)
            Ls.set_inputs(c0, in_np[:staged])
            while done < cycles:
                n = min(chunk, cycles - done)
                if staged < cycles:
                    n2 = min(chunk, cycles - staged)
                    Ls.set_inputs(c0 + staged, in_np[:n2])
                    staged += n2
                Ls.step(n, hashes=h_np[:n] if n == chunk else np.ascontiguousarray(h_np[:n]))
                done += n

        e2e_step()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 2))
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        barrier()
        el = D.max_over_ranks(el, dist)
        e2e = {"value": (total_lanes * n_replicas if single else total_lanes) * cycles * e2e_steps / el, "unit": UNIT,
               "h2d_bytes_per_step": int(cycles * circ.n_inputs * lanes * 8),
               "d2h_bytes_per_step": int(cycles * lanes * 8), "steps": e2e_steps,
               "path": "rs_set_inputs(host pinned, next chunk, copy stream) + rs_step_cycles(hashes=HOST) "
                       f"per chunk of {chunk} cycles (2-chunk ring)"}
        Ls.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        nl, nc = cpu_sample_plan(circ, 10.0, cores)
        rate, dt = oracle_rate(circ, cfg.stim_seed, nl, nc, threads=cores)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{nl} lanes x {nc} cycles of {args.config} ({dt:.2f} s)"}

    if rank == 0:
        scaling = "strong" if levelcut else "weak" if (single or args.scaling == "weak") else "strong"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "ms_per_step_median": med_ms,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u64",
            "data": "synthetic",
            "config": {"workload": workload(args.config, total_lanes, lanes, cycles, circ.n_ops, info["n_levels"],
                                            world, scaling, levelcut),
                       **({"level_cut_across_gpus": world} if levelcut else {}),
                       "lanes_total": total_lanes, "lanes_per_gpu": lanes, "cycles_per_step": cycles,
                       "hash": not args.no_hash,
                       "l2": "flushed (256 MB write) before every timed step",
                       "mode": "single" if single else "lanes", "launch": L.shape(),
                       "collective": "none on the data path (gloo barrier + max-over-ranks timing only)",
                       **({"devices": ndev} if world > 1 else {}),
                       **({"level_cut_parts": args.parts} if args.parts > 1 else {}),
                       **({"repcut_partitions": args.repcut} if args.repcut >= 1 else {}),
                       **({"l2_policy": args.l2_policy} if args.l2_policy else {}),
                       "state_bytes_per_gpu": info["state_bytes_per_lane"] * lanes,
                       "graph_passes": None if args.no_passes else {
                           "ops_evaluated": info["n_ops"], "aliases": info["n_alias"],
                           "folded": info["n_folded"], "mux_chains_counted": info["n_mux_chain"]},
                       **({"watched_signals": args.watch} if args.watch else {})},
            "op_evals_per_s": value * circ.n_ops,
            "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src, "alg_bytes_per_launch": alg_bytes,
                         "alg_bytes_per_lane_cycle": info["alg_bytes_per_lane_cycle"],
                         "alg_bytes_per_lane_cycle_without_passes": info0["alg_bytes_per_lane_cycle"],
                         "graph_alg_bytes": info["graph_alg_bytes"], "kernel": kernel_name},
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "step_ms": step_ms,
        }
        if hash_off:
            off_med = float(np.median(hash_off))
            line["hash_off"] = {"value": (total_lanes * n_replicas if single else total_lanes) * cycles / (off_med / 1e3),
                                "ms_per_step_median": off_med, "steps": len(hash_off),
                                "roofline_frac": alg_bytes / (off_med / 1e3) / 1e9 / peak}
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
