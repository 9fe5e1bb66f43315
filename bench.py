#!/usr/bin/env python3
"""Benchmark: QAOA Max-Cut levels/s and amplitude-updates/s on B200.

Workload (BASELINE.json configs[2], the roofline configuration; configs[1]
N=26 p=4 is a parity-test case): random 3-regular graph N=30 (seed 0),
p=10 levels with params_from_seed(10, 0) (reference bench.py:61-67), complex128
state of 16 GiB, launch-control init, fused <C>.  One "step" = one full
``simulate`` (p levels) + ``expectation`` with the graph and angles already on
the device.  The 16 GiB state is far larger than L2 (126 MB), so no flush is
needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--qubits 30] [--levels 10] [--exact] [--graph u3r|er]

N > 1 (one process per GPU via torch.distributed.run, NCCL): the same N=30
state is sharded over the G ranks by its top log2(G) qubits (strong scaling,
paper_2312_03019_b200.sharded: shard-local fused sweeps + one global<->local
chunk exchange per level).  ``--replicas`` instead runs one full state per rank
(weak scaling).  Device time is the max over ranks.

``--impl reference`` times the CPU oracle (oracle/, a C restatement of the
reference's algorithm, bit-exact with it) on all host threads at the same
config: each step is one level of the same N=30 p=10 circuit (~12 s on 16
threads), plus the cut-table build, expectation and a 1-thread sample.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QAOA layers/sec and amplitude-updates/sec at N qubits; % HBM roofline; 1/2/4/8 GPU"
L2_BYTES = 126 * 2**20


def l2_note(state_bytes, shards=1):
    """The timing-rule note on L2: no flush is needed when each GPU's state is
    far larger than the 126 MB L2 (every sweep streams it from HBM)."""
    per = state_bytes // shards
    if per >= 8 * L2_BYTES:
        return f"no flush: {per / 2**30:.3g} GiB state per GPU >> 126 MB L2"
    where = "L2-resident" if per <= L2_BYTES else "partly L2-resident"
    return f"not flushed: {per / 2**20:.4g} MiB state per GPU is {where} (not a headline size)"


UNIT = "layers/s"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world: int, local: int, backend: str = "nccl"):
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:  # test mode: several ranks may share one GPU; exchanges stage through host memory
        dist.init_process_group("gloo")
    return dist


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"  # /opt/skills/guides/B200_PROFILING.md fallback


def ncu_traffic(n: int):
    """dram read+write bytes per sweep launch from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        rec = d.get(str(n))
        return float(rec["dram_bytes_per_launch"]) if rec else None
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw,enforced.power.limit,clocks.mem")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw, lim, mem = [], 0.0, set(), [], [], []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
            for dst, i in ((pw, 6), (lim, 7), (mem, 8)):
                try:
                    dst.append(float(parts[i]))
                except (IndexError, ValueError):
                    pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
               "samples": len(sm)}
        if pw:
            out["power_w"] = statistics.median(pw)
        if lim:
            out["power_limit_w"] = statistics.median(lim)
        if mem:
            out["mem_mhz"] = statistics.median(mem)
        return out


def ref_graph_edges(n: int, graph: str):
    """The bench graph restated with the oracle's generators (the GPU box has no
    /root/reference): u3r seed 0 (graph.py:170-205; odd N: u3r(N-1) plus an
    isolated node) or ER(0.5) seed 0 (test_acceptance.py:46-57 pattern)."""
    from oracle import oracle as O

    if graph == "er":
        rng = np.random.default_rng(0)
        return [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.5]
    return O.random_regular_edges(n - (n % 2), 3, 0)


class RefLevels:
    """The reference's CPU path (oracle port: cost.py:162-176 + circuit.py:89-94,
    bit-exact with the reference) on the host, one QAOA level per call, cycling
    through the p levels of params_from_seed(p, 0); level 0 includes the
    launch-control init (circuit.py:42-48)."""

    def __init__(self, n: int, p: int, graph: str, threads: int):
        from oracle import oracle as O

        self.O, self.n, self.p, self.threads = O, n, p, threads
        edges = ref_graph_edges(n, graph)
        self.rm = O.row_masks(n, edges)
        self.E = len(edges)
        self.gm, self.bt = O.params_from_seed(p, 0)
        self.amps = np.empty(1 << n, dtype=np.complex128)
        self.level = 0

    def step(self) -> float:
        O, t0 = self.O, time.perf_counter()
        if self.level == 0:
            O.lib().orc_init_uniform(self.n, O._ptr(self.amps, O._f64p), self.threads)
        O.apply_cost(self.amps, self.n, self.rm, self.E, self.gm[self.level], threads=self.threads)
        O.apply_mixer(self.amps, self.n, self.bt[self.level], threads=self.threads)
        self.level = (self.level + 1) % self.p
        return time.perf_counter() - t0

    def cut_table_s(self) -> float:
        t0 = time.perf_counter()
        ct = self.O.cut_counts(self.n, self.rm, threads=self.threads)
        dt = time.perf_counter() - t0
        del ct
        return dt

    def expectation(self) -> tuple[float, float]:
        t0 = time.perf_counter()
        e = self.O.expectation(self.n, self.rm, self.amps, threads=self.threads)
        return e, time.perf_counter() - t0


def cpu_reference_level(n: int, p: int, graph: str, threads: int):
    """One level (init + cost + mixer) of the bench's own config on the host:
    the GPU line's bounded cpu_baseline sample (~12 s at N=30 on 16 threads)."""
    r = RefLevels(n, p, graph, threads)
    dt = r.step()
    del r
    return (n + 1) * (1 << n) / dt, dt


def single_thread_sample(n: int, graph: str, n_sample: int = 24):
    """T=1 beside T=all: one level at a bounded size."""
    n_sample = min(n, n_sample)
    r = RefLevels(n_sample, 1, graph, 1)
    dt = r.step()
    return {"threads": 1, "sample": f"1 level of the same graph family at N={n_sample}",
            "level_s": dt, "amp_updates_per_s": (n_sample + 1) * (1 << n_sample) / dt,
            "layers_per_s_at_N": (n_sample + 1) * (1 << n_sample) / dt / ((n + 1) * (1 << n))}


def run_reference(args, rank: int, world: int):
    """The reference arm: the reference's CPU path (oracle port) at the GPU
    line's own config (N, p, graph, angles), one QAOA level per step, all host
    threads.  Also times the cut-table build (cost.py:88-99, pre-warmed by the
    reference before its layers) and expectation (circuit.py:116-121) apart,
    and a single-thread sample."""
    if rank != 0:
        return 0
    from oracle import oracle as O

    O.lib()
    t_start = time.perf_counter()
    threads = len(os.sched_getaffinity(0))
    n, p = args.n, args.p
    per_level = (n + 1) * (1 << n)
    ref = RefLevels(n, p, args.graph, threads)
    table_s = ref.cut_table_s()
    for _ in range(args.warmup):
        ref.step()
    times = [ref.step() for _ in range(args.steps)]
    total = sum(times)
    e_val, expect_s = ref.expectation()
    complete = (args.warmup + args.steps) % p == 0
    t1 = single_thread_sample(n, args.graph)
    layers = args.steps / total
    wall = time.perf_counter() - t_start
    line = {
        "impl": "reference", "metric": METRIC, "value": layers, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": workload_name(args),
                   "n_qubits": n, "p": p, "graph": args.graph,
                   "schedule": "reference (cost layer + n RX per level, increasing qubit order)",
                   "parallelism": "host CPU, OpenMP",
                   "l2": l2_note(16 << n)},
        "step": "one QAOA level of the config's p-level circuit (levels cycle 0..p-1; "
                "level 0 includes the launch-control init)",
        "amp_updates_per_s": layers * per_level,
        "level_s": {"median": statistics.median(times), "min": min(times), "max": max(times)},
        "cut_table_build_s": table_s,
        "expectation_s": expect_s,
        "expectation": e_val if complete else None,
        "single_thread": t1,
        "cpu_baseline": {"value": layers, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} timed levels of the config itself "
                                   f"(N={n}, p={p}, {args.graph}) after {args.warmup} warm-up levels"},
        "e2e": {"value": layers, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "consistency": {"timed_s": total, "wall_s": wall},
    }
    print(json.dumps(line), flush=True)
    return 0


def sweep_kinds(L, n: int, p: int, exact: bool, count: int) -> list[str]:
    """Kind of every sweep of one qaoa_run_layers call, from the engine's own
    plan export (qaoa_plan: carry, q, pre-cost, stage 1, mid-cost, stage 2,
    exchange per sweep)."""
    if n < 12:
        return ["whole circuit in one CTA"] * count
    buf = (ctypes.c_int * (7 * 256))()
    ns = L.qaoa_plan(n, p, 1 if exact else 0, buf, 256)
    kinds = []
    for i in range(max(ns, 0)):
        carry, _q, _pre, _s1, mid = buf[7 * i:7 * i + 5]
        if i == 0:
            kinds.append("launch-control sweep (no load)")
        elif mid >= 0:
            kinds.append("merged level-boundary sweep")
        elif i == ns - 1:
            kinds.append("last sweep (+<C>)")
        elif carry == 12:
            kinds.append("low-set sweep S0")
        else:
            kinds.append("single high-set sweep")
    return kinds if len(kinds) == count else ["sweep"] * count


def dominant_kernel_text(L, n: int, p: int, exact: bool, dom) -> str:
    """Which kernel runs the dominant sweep kind (the policy of qaoa_sweep32.cu
    sweep32_eligible / qaoa_sweep_tma.cu sweep_impl for the plan's geometry)."""
    if not dom:
        return "fused sweeps"
    carry = None
    buf = (ctypes.c_int * (7 * 256))()
    ns = L.qaoa_plan(n, p, 1 if exact else 0, buf, 256)
    for i in range(1, max(ns, 0)):
        c, _q, _pre, _s1, mid = buf[7 * i:7 * i + 5]
        if ("merged" in dom and mid >= 0) or ("low-set" in dom and c == 12) or \
                ("last" in dom and i == ns - 1):
            carry = c
            break
    s32 = (not exact and carry is not None and 3 <= carry <= 7 and os.environ.get("QAOA_SWEEP32", "1") != "0"
           and (carry in (3, 7) or "merged" not in dom))
    if s32:
        ctas = "three" if ("merged" in dom and carry == 3) else "two"
        xch = "no exchange" if carry == 7 else ("two exchanges" if "merged" in dom else "one exchange")
        return (f"{dom}: qb::sweep32_kernel (128 threads x 32 amplitudes per 4096-amplitude tile, "
                f"{ctas} CTAs per SM, L2 tile prefetch; five-bit register windows, {xch}, "
                "no lane transposes; C = %d)" % carry)
    return (f"{dom}: qb::sweep_kernel (256 threads x 16 amplitudes per 4096-amplitude tile, two CTAs "
            "per SM, L2 tile prefetch)")


def p1_closed_form(n: int, edges, gamma: float, beta: float) -> float:
    """<C> of a p=1 circuit on any unweighted graph, edge by edge (Wang, Hadfield,
    Jiang, Rieffel 2018, mapped to the reference's convention).
    The check for states no CPU can hold (N=36 over 8 GPUs)."""
    adj = [set() for _ in range(n)]
    for i, j in edges:
        adj[i].add(j)
        adj[j].add(i)
    s2b, sb2 = math.sin(2 * beta), math.sin(beta) ** 2
    cg, c2g, sg = math.cos(gamma), math.cos(2 * gamma), math.sin(gamma)
    total = 0.0
    for u, v in edges:
        du, dv, lam = len(adj[u]) - 1, len(adj[v]) - 1, len(adj[u] & adj[v])
        total += 0.5 + 0.25 * s2b * sg * (cg ** du + cg ** dv) \
            - 0.25 * sb2 * cg ** (du + dv - 2 * lam) * (1 - c2g ** lam)
    return total


def closed_form_check(g, params, value):
    """p=1 runs: <C> against the closed form; raises past the 1e-10 contract."""
    if params.p != 1:
        return None
    cf = p1_closed_form(g.n, [(i, j) for i, j, _ in g.edges], params.gamma[0], params.beta[0])
    rel = abs(value - cf) / abs(cf)
    if rel > 1e-10:
        raise SystemExit(f"<C> = {value!r} differs from the p=1 closed form {cf!r} (rel {rel:.2e})")
    return {"value": cf, "rel_err": rel}


def make_graph(Q, args):
    if args.graph == "er":
        return Q.erdos_renyi_graph(args.n, 0.5, seed=0)
    if args.n % 2:  # no 3-regular graph on an odd node count: u3r(N-1) plus an isolated node
        base = Q.random_regular_graph(args.n - 1, 3, seed=0)
        return Q.Graph.from_edges(args.n, list(base.edges))
    return Q.random_regular_graph(args.n, 3, seed=0)


def workload_name(args) -> str:
    gname = ("u3r" if args.n % 2 == 0 else f"u3r({args.n - 1}) + isolated node") \
        if args.graph == "u3r" else "ER(0.5)"
    cfg = {("u3r", 30, 10): "BASELINE configs[2]", ("er", 33, 4): "BASELINE configs[3]",
           ("u3r", 26, 4): "BASELINE configs[1]", ("u3r", 20, 1): "BASELINE configs[0]"}
    tag = cfg.get((args.graph, args.n, args.p), "custom")
    return f"{gname} N={args.n} seed 0, p={args.p} levels, complex128 ({tag})"


def run_sharded(args, rank: int, world: int, local: int):
    """Strong scaling: one N-qubit state sharded over `world` GPUs (NCCL)."""
    import torch
    import torch.distributed as tdist

    import paper_2312_03019_b200 as Q
    from paper_2312_03019_b200 import _lib
    from paper_2312_03019_b200.sharded import (CudaShard, DistExchanger, IpcChunkExchanger,
                                               IpcExchanger, simulate_sharded,
                                               simulate_sharded_fused)

    if world & (world - 1):
        raise SystemExit("sharded mode needs a power-of-two GPU count")
    if args.share_device:
        local = 0
    dist = init_dist(world, local, args.dist_backend)
    torch.cuda.set_device(local)
    gbits = world.bit_length() - 1
    # strong: the --qubits state over the G GPUs; weak: 2^qubits amplitudes per GPU
    # (N = qubits + log2 G: 33@1 -> 36@8 at 128 GiB per GPU)
    n, p = (args.n + gbits if args.scaling == "weak" else args.n), args.p
    args.n = n
    g = make_graph(Q, args)
    params = Q.params_from_seed(p, 0)
    fused = args.exchange == "ipc"
    shard = CudaShard(n - gbits, rank, device=local, exact=args.exact,
                      stream=None if fused else torch.cuda.current_stream(local).cuda_stream)
    fallback = None
    exch = None
    if fused:
        try:
            exch = (IpcChunkExchanger(shard, rank, world, args.chunks) if args.chunks > 1
                    else IpcExchanger(shard, rank, world))
        except Exception as exc:  # no CUDA IPC / peer access between these GPUs
            fallback = f"CUDA IPC unavailable ({exc}); NCCL staging path used"
    ok = torch.tensor([0 if (fused and exch is None) else 1], dtype=torch.int32,
                      device="cpu" if args.dist_backend == "gloo" else f"cuda:{local}")
    tdist.all_reduce(ok, op=tdist.ReduceOp.MIN)
    if fused and int(ok.item()) == 0:  # every rank must take the same path
        if exch is not None and hasattr(exch, "close"):
            exch.close()
        fused, exch = False, None
        fallback = fallback or "a peer could not map CUDA IPC; NCCL staging path used"
        shard.close()
        shard = CudaShard(n - gbits, rank, device=local, exact=args.exact,
                          stream=torch.cuda.current_stream(local).cuda_stream)
    if exch is None:
        exch = DistExchanger(shard, rank, world)
    if hasattr(exch, "timing"):
        exch.timing = True  # CUDA events around every exchange kernel launch
    def step():
        if fused:
            simulate_sharded_fused(g, params, [shard], exch, gbits, exact=args.exact, expect=True)
        else:
            simulate_sharded(g, params, [shard], exch, gbits)
        dev = "cpu" if args.dist_backend == "gloo" else f"cuda:{local}"
        part = torch.tensor([shard.expectation()], dtype=torch.float64, device=dev)
        allp = [torch.zeros_like(part) for _ in range(world)]
        tdist.all_gather(allp, part)
        return float(sum(t.item() for t in allp))  # rank order: deterministic

    for _ in range(max(args.warmup, 3)):
        val = step()
    dist.barrier()
    torch.cuda.synchronize(local)
    if hasattr(exch, "exchange_ms"):
        exch.collect()
        exch.exchange_ms.clear()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    step_bytes = 0.0
    with ClockSampler(local) as clocks:
        t0 = time.perf_counter()
        start.record()
        for _ in range(args.steps):
            val = step()
            nl, hb = ctypes.c_int(), ctypes.c_double()
            _lib.load().qaoa_last_run_stats(shard.eng.ptr, ctypes.byref(nl), ctypes.byref(hb))
            launches += nl.value + (p * max(args.chunks, 1) if fused else 0)
            step_bytes = hb.value  # this rank's algorithmic sweep bytes per step
        stop.record()
        torch.cuda.synchronize(local)
        wall_s = time.perf_counter() - t0
    dev_ms = start.elapsed_time(stop)
    xms = None
    if getattr(exch, "exchange_ms", None) is not None:
        exch.collect()
        if exch.exchange_ms:
            xms = statistics.mean(exch.exchange_ms)
    tx = torch.tensor([xms if xms is not None else -1.0], dtype=torch.float64,
                      device="cpu" if args.dist_backend == "gloo" else f"cuda:{local}")
    tdist.all_reduce(tx, op=tdist.ReduceOp.MAX)
    xms = float(tx.item()) if tx.item() > 0 else None
    tw = torch.tensor([wall_s], dtype=torch.float64,
                      device="cpu" if args.dist_backend == "gloo" else f"cuda:{local}")
    tdist.all_reduce(tw, op=tdist.ReduceOp.MAX)
    wall_s = float(tw.item())
    t = torch.tensor([dev_ms], device="cpu" if args.dist_backend == "gloo" else f"cuda:{local}")
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    dev_ms = float(t.item())
    layers = p * args.steps / (dev_ms * 1e-3)
    per_level = (n + 1) * (1 << n)
    xbytes = (world - 1) / world * 16 * (1 << (n - gbits))  # per rank per direction per level
    step_s = dev_ms * 1e-3 / args.steps
    step_gbps = step_bytes / step_s / 1e9
    if rank == 0:
        peak, peak_kind = measured_peaks()
        line = {
            "metric": METRIC, "value": layers, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "c128",
            "data": "synthetic",
            "config": {"workload": workload_name(args),
                       "n_qubits": n, "p": p, "graph": args.graph,
                       "parallelism": f"state sharded over {world} GPUs (top {gbits} qubits), "
                       + (f"fused in-place exchange kernel over CUDA-IPC peer memory (NVLink P2P), "
                          f"pipelined with the sweeps in {args.chunks} chunks"
                          if fused else "NCCL P2P exchange + separate RX sweep"),
                       "l2": l2_note(16 << n, world)},
            "amp_updates_per_s": layers * per_level, "expectation": val,
            "test_mode": bool(args.share_device or args.dist_backend != "nccl"),
            "exchange_fallback": fallback,
            "nvlink": {"bytes_per_level_per_rank_per_direction": xbytes,
                       "peak_GBps_per_direction": 770.0,
                       "peak_kind": "measured 8-rank bus bandwidth (B200_PROFILING.md); "
                                    "900 GB/s nominal NVLink 5",
                       # per exchange: (G-1)/G of this rank's slice of 16 B x 2^n_local
                       # crosses NVLink in each direction; kernel time from CUDA
                       # events around every exchange launch, max over ranks
                       "exchange_ms": xms,
                       "achieved_GBps_per_direction": (xbytes / (xms * 1e-3) / 1e9) if xms else None,
                       "frac": (xbytes / (xms * 1e-3) / 1e9 / 770.0) if xms else None,
                       "exchanges_per_step": p,
                       # step-level: exchange bytes over the whole step time (the
                       # exchange overlaps the sweeps, so this is a lower bound)
                       "achieved_GBps_step_level": xbytes * p / step_s / 1e9},
            "closed_form_p1": closed_form_check(g, params, val),
            # step-level roofline: a rank's sweep bytes over the whole step,
            # exchange and peer waits included (no per-kernel split here: the
            # pipelined sweeps run as tile ranges interleaved with the exchange)
            "roofline": {"bound": "hbm", "achieved": step_gbps, "peak": peak, "unit": "GB/s",
                         "frac": step_gbps / peak, "traffic": None, "peak_kind": peak_kind,
                         "kernel": "step level: fused sweeps + in-place exchange (rank 0 bytes / "
                                   "max-over-ranks step time)",
                         "algorithmic_bytes_per_step": step_bytes},
            "cpu_baseline": None,
            # the sharded step is host-driven from host inputs (graph, angles ->
            # phase tables and relabelled masks every level) to <C> on the host
            "e2e": {"value": p * args.steps / wall_s, "unit": UNIT,
                    "h2d_bytes_per_step": int(p * (16 * (g.tot_edge + 1) * 2 + 16) + 8 * n * (p + 1)),
                    "d2h_bytes_per_step": 8,
                    "api": "paper_2312_03019_b200.sharded.simulate_sharded_fused + sharded_expectation"},
            "gpu_launches": launches, "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if hasattr(exch, "close"):
        tdist.barrier()  # every rank is done with the peers' shards ...
        exch.close()
        tdist.barrier()  # ... and has unmapped them before any shard is freed
    shard.close()
    dist.destroy_process_group()
    return 0


def run_ours(args, rank: int, world: int, local: int):
    import torch

    import paper_2312_03019_b200 as Q
    from paper_2312_03019_b200 import _lib

    dist = init_dist(world, local)
    device = local if world > 1 else 0
    torch.cuda.set_device(device)
    n, p = args.n, args.p
    g = make_graph(Q, args)
    params = Q.params_from_seed(p, 0)  # same RNG stream as reference bench.py:61-67
    tables, cs, ss = Q.level_arrays(g, params)
    stream = torch.cuda.Stream(device)
    eng = Q.Engine(n, device, stream=stream.cuda_stream)
    if args.e2e_steps is None:  # same step count as the device-timed loop
        args.e2e_steps = args.steps
    eng.ensure_graph(g)
    flags = _lib.RUN_EXPECTATION | _lib.RUN_TIMING | (_lib.RUN_EXACT if args.exact else 0)
    L = _lib.load()

    def step():
        eng.call("qaoa_run_layers", p, _lib.dptr(tables.view(np.float64)), _lib.dptr(cs),
                 _lib.dptr(ss), flags)

    for _ in range(max(args.warmup, 3)):
        step()
    expect_val = eng.scalar("qaoa_expectation")

    # ---- device-timed region: K steps, events on the engine's stream -------
    if dist:
        dist.barrier()
    torch.cuda.synchronize(device)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launch_ms: list[float] = []
    launches = 0
    with ClockSampler(device) as clocks:
        start.record(stream)
        for _ in range(args.steps):
            step()
            buf = (ctypes.c_float * 4096)()
            k = L.qaoa_layer_timings(eng.ptr, buf, 4096)
            launch_ms.extend(buf[:k])
            nl, hb = ctypes.c_int(), ctypes.c_double()
            L.qaoa_last_run_stats(eng.ptr, ctypes.byref(nl), ctypes.byref(hb))
            launches += nl.value
        stop.record(stream)
        torch.cuda.synchronize(device)
    if dist:
        dist.barrier()
    dev_ms = start.elapsed_time(stop)
    if dist:
        t = torch.tensor([dev_ms], device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
    layers_per_s = world * p * args.steps / (dev_ms * 1e-3)
    per_level = (n + 1) * (1 << n)
    sweep_bytes = hb.value  # algorithmic bytes of the last step's sweeps
    sweeps_per_step = len(launch_ms) // max(args.steps, 1)

    # ---- roofline of the dominant kernel: the sweeps of one step classified by
    # the engine's own plan (qaoa_plan), the kind with the largest share of the
    # step is the line's `roofline`; the all-sweeps average is kept beside it ----
    peak, peak_kind = measured_peaks()
    step_sweep_ms = sum(launch_ms) / max(args.steps, 1)
    achieved = sweep_bytes / (step_sweep_ms * 1e-3) / 1e9
    traffic = ncu_traffic(n)
    r_star = 1 + -(-max(0, n - 13) // 10)
    last = launch_ms[-sweeps_per_step:]
    kinds = sweep_kinds(L, n, p, args.exact, len(last))
    per_kind = {}
    for kind, ms in zip(kinds, last):
        d = per_kind.setdefault(kind, {"launches_per_step": 0, "ms": 0.0})
        d["launches_per_step"] += 1
        d["ms"] += ms
    for kind, d in per_kind.items():
        b = (16 if kind.startswith("launch-control") else 32) * (1 << n)
        d["avg_ms"] = d["ms"] / d["launches_per_step"]
        d["share"] = d["ms"] / sum(last)
        d["GBps"] = b / (d["avg_ms"] * 1e-3) / 1e9
        d["frac"] = d["GBps"] / peak
        d["algorithmic_bytes_per_launch"] = b
    dom = max(per_kind, key=lambda k: per_kind[k]["ms"]) if per_kind else None
    dk = per_kind.get(dom, {"GBps": achieved, "frac": achieved / peak, "avg_ms": None,
                            "algorithmic_bytes_per_launch": 32 * (1 << n)})
    roofline = {"bound": "hbm", "achieved": dk["GBps"], "peak": peak, "unit": "GB/s",
                "frac": dk["frac"], "traffic": traffic if dom and "merged" in dom else None,
                "peak_kind": peak_kind,
                "kernel": dominant_kernel_text(L, n, p, args.exact, dom),
                "algorithmic_bytes_per_launch": dk["algorithmic_bytes_per_launch"],
                "avg_launch_ms": dk["avg_ms"],
                "per_kind": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv)
                                 for kk, vv in d.items()} for k, d in per_kind.items()},
                # every sweep of the step together (21 at N=30 p=10)
                "all_sweeps": {"achieved": achieved, "frac": achieved / peak,
                               "avg_launch_ms": step_sweep_ms / max(sweeps_per_step, 1),
                               "launches_per_step": sweeps_per_step},
                "launch_ms_last_step": [round(x, 3) for x in last],
                # whole-step figures against B_alg = 32 R* 2^N per
                # level (R* = sweeps of a 2^13 tile) and against the one-pass floor
                "r_star": r_star,
                "level_roofline_frac_Rstar": (32 * r_star * (1 << n) * p
                                              / (dev_ms / args.steps * 1e-3)) / 1e9 / peak,
                "level_floor_frac": (32 * (1 << n) * p / (dev_ms / args.steps * 1e-3)) / 1e9 / peak}

    # ---- K1, the cut-table builder, timed once --------
    cut_table = None
    if args.cut_table:
        eng.call("qaoa_build_cut_table")  # warm-up (module load, allocation)
        # CUDA events around the kernel launch inside the library (the host's
        # launch latency is not part of the kernel's time); median of 5 builds
        k1 = []
        for _ in range(5):
            eng.call("qaoa_build_cut_table")
            buf = (ctypes.c_float * 4)()
            L.qaoa_layer_timings(eng.ptr, buf, 4)
            k1.append(buf[0])
        ms = statistics.median(k1)
        bpe = 1 if g.tot_edge <= 255 else 2
        gbps = (bpe << n) / (ms * 1e-3) / 1e9
        cut_table = {"kernel": "qb::cut_table_warp_kernel (K1, SURVEY 8a a3: cost.py:88-99)",
                     "ms": ms, "states_per_s": (1 << n) / (ms * 1e-3),
                     "bytes_written": bpe << n, "GBps": gbps, "dtype": "uint8" if bpe == 1 else "uint16",
                     # K1's roofline is its table write, w_C 2^N bytes
                     "roofline_frac": gbps / peak}
        eng.call("qaoa_free_cut_table")

    # ---- end to end through the public API: host inputs -> <C> on the host ----
    e2e = None
    if args.e2e_steps > 0:
        s = Q.StateVector(n, engine=eng)
        torch.cuda.synchronize(device)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            # host -> device: graph masks + phase tables + RX coefficients (pinned)
            eng.graph_key = None
            sv = Q.simulate(g, params, "bitwise", max_qubits=n, state=s, exact=args.exact)
            val = Q.expectation(g, sv)  # device -> host: <C>
        e2e_s = time.perf_counter() - t0
        if dist:
            t = torch.tensor([e2e_s], device=f"cuda:{device}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        h2d = 8 * n + tables.nbytes + cs.nbytes + ss.nbytes
        e2e = {"value": world * p * args.e2e_steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 8,
               "api": "paper_2312_03019_b200.simulate + expectation",
               # a separate loop of the same K steps (wall clock, host inputs,
               # every step synchronous): the same kernels as `value`
               "steps": args.e2e_steps}
        assert abs(val - expect_val) <= 1e-10 * abs(expect_val)

    # ---- symmetric half-state mode (opt-in API mode, NOT the headline): the
    # same circuit on the 2^(N-1)-amplitude half, psi(x) == psi(~x) ----------
    sym = None
    if (args.symmetric_probe and world == 1 and n >= 13 and g.is_unweighted and not args.exact
            and torch.cuda.mem_get_info(device)[0] > (16 << (n - 1)) + (4 << 30)):
        from paper_2312_03019_b200.symmetric import simulate_symmetric

        ss = simulate_symmetric(g, params)
        for _ in range(max(args.warmup, 3) - 1):
            simulate_symmetric(g, params, state=ss)
        torch.cuda.synchronize(device)
        sym_launch: list[float] = []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            simulate_symmetric(g, params, state=ss, timing=True)
            e_sym = Q.expectation(g, ss)
            buf = (ctypes.c_float * 4096)()
            k = L.qaoa_layer_timings(ss.half_engine.ptr, buf, 4096)
            sym_launch.extend(buf[:k])
        sym_s = time.perf_counter() - t0
        per_step = len(sym_launch) // max(args.steps, 1)
        sym_dev_ms = sum(sym_launch) / max(args.steps, 1)
        sym = {"value": p * args.steps / sym_s, "unit": UNIT, "ms_per_step": 1e3 * sym_s / args.steps,
               "timing": "wall clock over K steps through simulate(..., symmetric=True) + "
                         "expectation (one qaoa_run_layers call per step, <C> read back)",
               "device_ms_per_step": sym_dev_ms,
               "launch_ms_last_step": [round(x, 3) for x in sym_launch[-per_step:]],
               "schedule": "fast; mirror low set (stored blocks u and ~u = virtual qubits 0..10 "
                           f"and {n - 1} in one sweep), high sets on qubits 11..{n - 2}",
               "state": f"2^{n - 1} amplitudes (the x_{n - 1} = 0 half; psi(x) == psi(~x) bit for "
                        "bit), simulate(..., symmetric=True); not the headline",
               "expectation": e_sym, "expectation_rel_diff": abs(e_sym - expect_val) / abs(expect_val)}
        ss.half_engine.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = len(os.sched_getaffinity(0))
            rate, dt = cpu_reference_level(n, p, args.graph, threads)
            cpu = {"value": rate / per_level, "unit": UNIT, "cores": threads, "kind": "port",
                   "sample": f"level 1 (init + cost + mixer) of this config (N={n}, {args.graph}) "
                             f"on the oracle (C port of the reference path, {threads} OpenMP "
                             f"threads, {dt:.1f} s)",
                   "amp_updates_per_s": rate}
        except Exception as exc:  # the CPU baseline must never sink the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port", "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": layers_per_s, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            # N=1 is the base point of the --gpus N curve (default: strong, the
            # same N-qubit state sharded over more GPUs)
            "scaling": args.scaling, "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": workload_name(args),
                       "n_qubits": n, "p": p, "graph": args.graph,
                       "schedule": "exact" if args.exact else "fast",
                       "parallelism": "replicas" if world > 1 else "single",
                       "l2": l2_note(16 << n)},
            "amp_updates_per_s": layers_per_s * per_level,
            "expectation": expect_val,
            "closed_form_p1": closed_form_check(g, params, expect_val),
            "cut_table_build": cut_table,
            "symmetric_mode": sym,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        cl = line["clocks"]
        if cl.get("power_w"):
            # the sweeps run at the board power limit: energy per level is the
            # figure that time follows
            line["energy_j_per_level"] = cl["power_w"] * (dev_ms / args.steps) * 1e-3 / p
        print(json.dumps(line), flush=True)
    eng.close()
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--qubits", dest="n", type=int, default=30)
    ap.add_argument("--graph", choices=["u3r", "er"], default="u3r",
                    help="u3r = random 3-regular seed 0 (configs 0-2, 4); er = G(n, 0.5) seed 0 "
                         "(configs[3], the dense N=33 cut-table stress case)")
    ap.add_argument("--levels", dest="p", type=int, default=10)
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="end-to-end loop steps (default: --steps)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-symmetric-probe", dest="symmetric_probe", action="store_false",
                    help="skip the symmetric half-state mode measurement (reported beside the "
                         "headline, never as it)")
    ap.add_argument("--no-cut-table", dest="cut_table", action="store_false",
                    help="skip timing the K1 cut-table builder")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo = test mode (exchanges staged through host memory)")
    ap.add_argument("--share-device", action="store_true",
                    help="test mode: every rank uses cuda:0 (correctness of the sharded path "
                         "on a one-GPU box; not a performance number)")
    ap.add_argument("--exchange", choices=["ipc", "nccl"], default="ipc",
                    help="sharded runs: fused exchange kernel over CUDA-IPC peer pointers "
                         "(default) or the NCCL P2P staging path")
    ap.add_argument("--chunks", type=int, default=4,
                    help="sharded ipc runs: pipeline each exchange with the sweeps around it "
                         "in this many chunks (1 = no overlap)")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="N>1: strong = the --qubits state sharded over the GPUs; weak = "
                         "2^qubits amplitudes per GPU (N = qubits + log2 GPUs), e.g. "
                         "--qubits 33 --scaling weak: 33@1 .. 36@8")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: one full state per rank (weak scaling) instead of sharding")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1 and not args.replicas:
        return run_sharded(args, rank, world, local)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
