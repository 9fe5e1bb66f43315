"""Sharded (multi-GPU) host logic on CPU: qubit layout bookkeeping, the
global<->local chunk exchange over torch.distributed (gloo, world sizes 2 and
4) and in-process virtual shards, driven with oracle-backed CPU shards and
compared against the unsharded oracle (amplitudes <= 1e-12, <C> <= 1e-10 rel).
The same driver runs CUDA shards over NCCL (tests/test_gpu_sharded.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2312_03019_b200 as Q
from paper_2312_03019_b200.sharded import (
    DistExchanger,
    LocalExchanger,
    ShardLayout,
    gather_true_state,
    sharded_expectation,
    simulate_sharded,
)


def test_layout_swap_roundtrip():
    L = ShardLayout(10, 2)
    L.swap_top()
    assert L.phys[6:10] == [8, 9, 6, 7]
    assert L.swap_bits(1 << 6) == 1 << 8 and L.swap_bits(1 << 9) == 1 << 7
    x = 0b11_01_000000
    assert L.swap_bits(L.swap_bits(x)) == x
    L.swap_top()
    assert L.phys == list(range(10))
    g = Q.random_regular_graph(10, 3, seed=1)
    L.swap_top()
    masks = L.physical_row_masks(g)
    assert sum(bin(m).count("1") for m in masks) == g.tot_edge


def reference_state(g, pr):
    from oracle import oracle as O

    return O.simulate(g.n, g.row_mask, g.tot_edge, pr.gamma, pr.beta, threads=1)


@pytest.mark.parametrize("n,gbits,p", [(8, 1, 2), (10, 2, 3), (12, 3, 2), (13, 2, 4)])
def test_virtual_shards_cpu(n, gbits, p):
    from oracle.oracle import OracleShard

    g = Q.random_regular_graph(n, 3, seed=n) if n % 2 == 0 else Q.erdos_renyi_graph(n, 0.4, n)
    pr = Q.params_from_seed(p, n)
    G = 1 << gbits
    shards = [OracleShard(n - gbits, r) for r in range(G)]
    layout = simulate_sharded(g, pr, shards, LocalExchanger(shards), gbits)
    stored = np.concatenate([s.tensor().numpy() for s in shards])
    true = gather_true_state(layout, stored, 0)
    ref = reference_state(g, pr)
    assert np.max(np.abs(true - ref)) <= 1e-12
    from oracle import oracle as O

    e = sharded_expectation(shards)
    assert e == pytest.approx(O.expectation(n, g.row_mask, ref), rel=1e-10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, gbits, p, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import OracleShard

        g = Q.random_regular_graph(n, 3, seed=7)
        pr = Q.params_from_seed(p, 3)
        shard = OracleShard(n - gbits, rank)
        layout = simulate_sharded(g, pr, [shard], DistExchanger(shard, rank, world, piece_elems=64),
                                  gbits)

        def world_sum(parts):
            allp = [None] * world
            dist.all_gather_object(allp, parts)
            merged = {}
            for d in allp:
                merged.update(d)
            return merged

        e = sharded_expectation([shard], world_sum)
        shards = [torch.zeros_like(shard.tensor()) for _ in range(world)]
        dist.all_gather(shards, shard.tensor())
        if rank == 0:
            stored = np.concatenate([t.numpy() for t in shards])
            out.put((gather_true_state(layout, stored, 0), e))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,p", [(2, 10, 3), (4, 12, 2)])
def test_gloo_sharded_matches_unsharded(world, n, p):
    gbits = world.bit_length() - 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, gbits, p, q)) for r in range(world)]
    for pr_ in procs:
        pr_.start()
    true, e = q.get(timeout=120)
    for pr_ in procs:
        pr_.join(timeout=120)
        assert pr_.exitcode == 0
    g = Q.random_regular_graph(n, 3, seed=7)
    pr = Q.params_from_seed(p, 3)
    ref = reference_state(g, pr)
    assert np.max(np.abs(true - ref)) <= 1e-12
    from oracle import oracle as O

    assert e == pytest.approx(O.expectation(n, g.row_mask, ref), rel=1e-10)


# ---- the fused path (segmented runs + in-place exchange with RX of the
# arriving qubits): host driver against the oracle, exchange restated in numpy
class NumpyExchanger:
    """In-process stand-in for PeerExchanger: oracle.fused_exchange_numpy over
    the G oracle shards' arrays."""

    def __init__(self, shards):
        self.shards = shards

    def exchange(self, g_bits, p0, rx, factor):
        from oracle.oracle import fused_exchange_numpy

        assert factor[0] == 1.0 and factor[1] == 0.0  # oracle shards run exact levels
        fused_exchange_numpy([s.tensor().numpy() for s in self.shards], g_bits, p0, rx)


class GatherExchanger:
    """Multi-process stand-in for IpcExchanger over gloo: gather every shard,
    run the same in-place exchange, keep this rank's shard."""

    def __init__(self, shard, rank, world):
        self.shard, self.rank, self.world = shard, rank, world

    def exchange(self, g_bits, p0, rx, factor):
        from oracle.oracle import fused_exchange_numpy

        parts = [torch.zeros_like(self.shard.tensor()) for _ in range(self.world)]
        dist.all_gather(parts, self.shard.tensor())
        arrs = [t.numpy().copy() for t in parts]
        fused_exchange_numpy(arrs, g_bits, p0, rx)
        self.shard.tensor().numpy()[:] = arrs[self.rank]


def test_layout_swap_at_p0():
    L = ShardLayout(16, 2)
    p0 = 10
    L.swap_at(p0)
    assert L.phys[10:12] == [14, 15] and L.phys[14:16] == [10, 11]
    assert L.swap_bits(1 << 10, p0) == 1 << 14 and L.swap_bits(1 << 15, p0) == 1 << 11
    x = 0b10_0000_11_0000000000
    assert L.swap_bits(L.swap_bits(x, p0), p0) == x


def test_fused_exchange_numpy_is_transpose_plus_rx():
    """The numpy restatement moves (shard r, local (y, h)) to (shard h, local (y, r))
    and with c = 1, s = 0 does nothing else."""
    from oracle.oracle import fused_exchange_numpy

    G, n, p0, g = 4, 8, 3, 2
    rng = np.random.default_rng(0)
    arrs = [rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n) for _ in range(G)]
    old = [a.copy() for a in arrs]
    fused_exchange_numpy(arrs, g, p0, np.array([1.0, 0.0, 0.0]))
    for r in range(G):
        for x in range(1 << n):
            h = (x >> p0) & (G - 1)
            y_lo, y_hi = x & ((1 << p0) - 1), x >> (p0 + g)
            dst = y_lo | (r << p0) | (y_hi << (p0 + g))
            assert arrs[h][dst] == old[r][x]


@pytest.mark.parametrize("n,gbits,p", [(13, 1, 3), (14, 2, 2), (15, 3, 2)])
def test_fused_virtual_shards_cpu(n, gbits, p):
    from oracle import oracle as O
    from oracle.oracle import OracleShard
    from paper_2312_03019_b200.sharded import simulate_sharded_fused

    g = Q.random_regular_graph(n, 3, seed=n + 1) if n % 2 == 0 else Q.erdos_renyi_graph(n, 0.4, n)
    pr = Q.params_from_seed(p, n)
    shards = [OracleShard(n - gbits, r) for r in range(1 << gbits)]
    layout = simulate_sharded_fused(g, pr, shards, NumpyExchanger(shards), gbits, exact=True)
    stored = np.concatenate([s.tensor().numpy() for s in shards])
    true = gather_true_state(layout, stored, 0)
    ref = reference_state(g, pr)
    assert np.max(np.abs(true - ref)) <= 1e-12
    # one swap per level: an odd level count leaves S_0's top qubits global
    assert (layout.phys != list(range(n))) == (p % 2 == 1)
    assert sharded_expectation(shards) == pytest.approx(O.expectation(n, g.row_mask, ref),
                                                        rel=1e-10)


def _fused_worker(rank, world, port, n, gbits, p, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import OracleShard
        from paper_2312_03019_b200.sharded import simulate_sharded_fused

        g = Q.random_regular_graph(n, 3, seed=5)
        pr = Q.params_from_seed(p, 4)
        shard = OracleShard(n - gbits, rank)
        layout = simulate_sharded_fused(g, pr, [shard], GatherExchanger(shard, rank, world), gbits,
                                        exact=True)
        parts = [None] * world
        dist.all_gather_object(parts, {rank: shard.expectation()})
        merged = {}
        for d in parts:
            merged.update(d)
        e = float(sum(merged[r] for r in sorted(merged)))
        shards = [torch.zeros_like(shard.tensor()) for _ in range(world)]
        dist.all_gather(shards, shard.tensor())
        if rank == 0:
            stored = np.concatenate([t.numpy() for t in shards])
            out.put((gather_true_state(layout, stored, 0), e))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,p", [(2, 14, 3), (4, 14, 2)])
def test_gloo_fused_sharded_matches_unsharded(world, n, p):
    gbits = world.bit_length() - 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, n, gbits, p, q))
             for r in range(world)]
    for pr_ in procs:
        pr_.start()
    true, e = q.get(timeout=180)
    for pr_ in procs:
        pr_.join(timeout=120)
        assert pr_.exitcode == 0
    g = Q.random_regular_graph(n, 3, seed=5)
    pr = Q.params_from_seed(p, 4)
    ref = reference_state(g, pr)
    assert np.max(np.abs(true - ref)) <= 1e-12
    from oracle import oracle as O

    assert e == pytest.approx(O.expectation(n, g.row_mask, ref), rel=1e-10)


# ---- the pipelined schedule's host logic (no GPU): every sweep covers all its
# tiles exactly once, chunked sweeps only around exchanges, ordered correctly
class _PlanShard:
    """Stand-in shard exposing a synthetic plan (segment, carry, q, ntiles)."""

    def __init__(self, plan, exchanges, log, rank=0, n=24):
        self.plan, self.exchanges, self.log, self.rank, self.n = plan, exchanges, log, rank, n

    def sweep_info(self, i):
        return self.plan[i] if i < len(self.plan) else None

    def exchange_info(self, k):
        return (k, np.zeros(3), np.array([1.0, 0.0])) if k in self.exchanges else None

    def run_sweep_range(self, i, lo, cnt):
        self.log.append(("sweep", self.rank, i, lo, cnt))


class _LogExchanger:
    def __init__(self, log, n_chunks):
        self.log, self.n_chunks = log, n_chunks

    def after_pre_chunk(self, t):
        self.log.append(("pre", t))

    def sync_point(self):
        self.log.append(("sync",))

    def launch_chunks(self, g_bits, p0, rx, factor):
        self.log.append(("exchange",))

    def wait_chunk(self, r, t):
        self.log.append(("wait", r, t))


@pytest.mark.parametrize("chunks", [2, 4, 8])
def test_pipelined_schedule_covers_every_tile_once(chunks):
    from paper_2312_03019_b200.sharded import _run_pipelined

    nl, nt = 27, 1 << 15
    # 3 local sets at n_local = 27: S0 (carry 12), S1 (carry 4, q 12), S2 (top: carry 5, q 20)
    S0, S1, S2 = (12, 0), (4, 12), (5, 20)
    segs = [[S1, S0], [S2, S2, S0], [S1, S1, S0], [S2]]   # exchange after each S0
    plan = [(k, c, q, nt) for k, seg in enumerate(segs) for (c, q) in seg]
    log = []
    shards = [_PlanShard(plan, {0, 1, 2}, log, r) for r in range(2)]
    relabels = []
    _run_pipelined(shards, _LogExchanger(log, chunks), len(segs), 1, 11, nl,
                   lambda: relabels.append(len(log)))
    for r in range(2):
        done = {}
        for ev in log:
            if ev[0] == "sweep" and ev[1] == r:
                _, _, i, lo, cnt = ev
                done.setdefault(i, []).append((lo, cnt))
        assert sorted(done) == list(range(len(plan)))
        for i, rs in done.items():
            rs.sort()
            assert rs[0][0] == 0 and sum(c for _, c in rs) == nt
            assert all(a[0] + a[1] == b[0] for a, b in zip(rs, rs[1:]))
            if len(rs) > 1:  # only S0 (before an exchange) and non-top sweeps after one split
                assert plan[i][1:3] in (S0, S1)
    # one exchange per S0, each after all pre chunks and followed by the relabel
    ex = [j for j, ev in enumerate(log) if ev == ("exchange",)]
    assert len(ex) == 3 and len(relabels) == 3
    for j, rl in zip(ex, relabels):
        assert rl > j
        pre = [ev[1] for ev in log[:j] if ev[0] == "pre"]
        assert pre.count(chunks - 1) >= 1
