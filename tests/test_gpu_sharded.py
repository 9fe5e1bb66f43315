"""The sharded engine on the GPU: G virtual CUDA shards on one device (engine
contexts with x_hi = rank << n_local, device-to-device chunk exchange) against
the unsharded engine and the oracle.  Covers the fast-mode complement
bookkeeping across exchanges (beta values that select the second RX form)."""

import numpy as np
import pytest
import torch

import paper_2312_03019_b200 as Q
from paper_2312_03019_b200.sharded import (
    CudaShard,
    LocalExchanger,
    gather_true_state,
    sharded_expectation,
    simulate_sharded,
)

pytestmark = pytest.mark.gpu


def run_virtual(g, pr, gbits, exact=False):
    G = 1 << gbits
    shards = [CudaShard(g.n - gbits, r, exact=exact) for r in range(G)]
    layout = simulate_sharded(g, pr, shards, LocalExchanger(shards), gbits)
    e = sharded_expectation(shards)
    cmask = shards[0].get_cmask()
    assert all(s.get_cmask() == cmask for s in shards)
    stored = np.concatenate([s.tensor().cpu().numpy() for s in shards])
    for s in shards:
        s.close()
    return gather_true_state(layout, stored, cmask), e


@pytest.mark.parametrize("n,gbits,betas", [
    (16, 1, (0.4, 1.1)),
    (20, 2, (0.3, 2.9, 1.0)),      # second RX form on level 2
    (22, 3, (2.95, 3.05)),         # second form twice
    (24, 3, (0.8, 2.2, 3.0, 0.1)),
    (21, 2, (1.3,)),
])
def test_virtual_shards_match_unsharded(oracle, n, gbits, betas):
    g = Q.random_regular_graph(n, 3, seed=n) if n % 2 == 0 else Q.erdos_renyi_graph(n, 0.3, n)
    gammas = tuple(0.2 + 0.9 * k for k in range(len(betas)))
    pr = Q.QaoaParams(gammas, betas)
    ref = oracle.simulate(n, g.row_mask, g.tot_edge, gammas, betas)
    eref = oracle.expectation(n, g.row_mask, ref)
    for exact in (False, True):
        true, e = run_virtual(g, pr, gbits, exact=exact)
        assert np.max(np.abs(true - ref)) <= 1e-12, (n, gbits, exact)
        assert e == pytest.approx(eref, rel=1e-10)


def test_virtual_shards_config_c3_strong(oracle):
    """u3r N=28, p=3 over G=8 virtual shards vs the unsharded engine (device)."""
    n = 28
    g = Q.random_regular_graph(n, 3, seed=0)
    pr = Q.params_from_seed(3, 0)
    full = Q.simulate(g, pr, "bitwise", max_qubits=n)
    e_full = Q.expectation(g, full)
    ref = full.amps
    true, e = run_virtual(g, pr, 3)
    assert np.max(np.abs(true - ref)) <= 1e-12
    assert e == pytest.approx(e_full, rel=1e-10)


# ---- the fused path: segmented shard runs + in-place exchange kernel with the
# arriving qubits' RX (qaoa_exchange), G virtual shards on one device
def run_virtual_fused(g, pr, gbits, exact=False, expect=True):
    from paper_2312_03019_b200.sharded import PeerExchanger, simulate_sharded_fused

    G = 1 << gbits
    shards = [CudaShard(g.n - gbits, r, exact=exact) for r in range(G)]
    layout = simulate_sharded_fused(g, pr, shards, PeerExchanger(shards), gbits, exact=exact,
                                    expect=expect)
    e = sharded_expectation(shards)
    cmask = shards[0].get_cmask()
    assert all(s.get_cmask() == cmask for s in shards)
    stored = np.concatenate([s.tensor().cpu().numpy() for s in shards])
    for s in shards:
        s.close()
    return gather_true_state(layout, stored, cmask), e


@pytest.mark.parametrize("n,gbits,betas", [
    (14, 1, (0.4, 1.1)),
    (16, 2, (0.3, 2.9, 1.0)),      # second RX form on level 2
    (18, 3, (2.95, 3.05)),         # second form twice
    (22, 3, (0.8, 2.2, 3.0, 0.1)),
    (25, 2, (1.3, 0.7, 2.6)),      # 3 local sets + merges
    (24, 4, (2.0, 0.5)),           # 16 virtual shards
])
def test_fused_virtual_shards_match_oracle(oracle, n, gbits, betas):
    g = Q.random_regular_graph(n, 3, seed=n) if n % 2 == 0 else Q.erdos_renyi_graph(n, 0.3, n)
    gammas = tuple(0.2 + 0.9 * k for k in range(len(betas)))
    pr = Q.QaoaParams(gammas, betas)
    ref = oracle.simulate(n, g.row_mask, g.tot_edge, gammas, betas)
    eref = oracle.expectation(n, g.row_mask, ref)
    for exact in (False, True):
        true, e = run_virtual_fused(g, pr, gbits, exact=exact)
        assert np.max(np.abs(true - ref)) <= 1e-12, (n, gbits, exact)
        assert e == pytest.approx(eref, rel=1e-10)


def test_fused_virtual_shards_config_c3(oracle):
    """u3r N=30, p=4 over G=8 virtual shards (27 local qubits, 3 sets) vs the
    unsharded engine on the same device."""
    n = 30
    g = Q.random_regular_graph(n, 3, seed=0)
    pr = Q.params_from_seed(4, 0)
    full = Q.simulate(g, pr, "bitwise", max_qubits=n)
    e_full = Q.expectation(g, full)
    ref = full.amps
    del full
    true, e = run_virtual_fused(g, pr, 3)
    assert np.max(np.abs(true - ref)) <= 1e-12
    assert e == pytest.approx(e_full, rel=1e-10)


# ---- pipelined: exchange chunks overlapped with the sweeps before / after
def run_virtual_pipelined(g, pr, gbits, chunks, exact=False):
    from paper_2312_03019_b200.sharded import PeerChunkExchanger, simulate_sharded_fused

    G = 1 << gbits
    shards = [CudaShard(g.n - gbits, r, exact=exact) for r in range(G)]
    layout = simulate_sharded_fused(g, pr, shards, PeerChunkExchanger(shards, chunks), gbits,
                                    exact=exact, expect=True)
    e = sharded_expectation(shards)
    cmask = shards[0].get_cmask()
    stored = np.concatenate([s.tensor().cpu().numpy() for s in shards])
    for s in shards:
        s.close()
    return gather_true_state(layout, stored, cmask), e


@pytest.mark.parametrize("n,gbits,chunks,betas", [
    (14, 1, 2, (0.4, 1.1, 2.9)),     # 2 local sets, one-sweep segments
    (18, 2, 4, (0.3, 2.9, 1.0)),
    (24, 3, 4, (2.95, 3.05, 0.7)),   # 3 local sets: the sweep after X is the top set (whole)
    (27, 2, 8, (0.8, 2.2, 3.0, 0.1)),  # 3 local sets, 8 chunks
    (25, 1, 4, (1.3, 0.6)),          # 4 local sets: both sides of X pipelined
])
def test_pipelined_virtual_shards_match_oracle(oracle, n, gbits, chunks, betas):
    g = Q.random_regular_graph(n, 3, seed=n) if n % 2 == 0 else Q.erdos_renyi_graph(n, 0.3, n)
    gammas = tuple(0.2 + 0.9 * k for k in range(len(betas)))
    pr = Q.QaoaParams(gammas, betas)
    ref = oracle.simulate(n, g.row_mask, g.tot_edge, gammas, betas)
    eref = oracle.expectation(n, g.row_mask, ref)
    for exact in (False, True):
        true, e = run_virtual_pipelined(g, pr, gbits, chunks, exact=exact)
        assert np.max(np.abs(true - ref)) <= 1e-12, (n, gbits, chunks, exact)
        assert e == pytest.approx(eref, rel=1e-10)
