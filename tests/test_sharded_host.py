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
