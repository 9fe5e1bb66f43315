"""Symmetric half-state mode (paper_2312_03019_b200.symmetric): N qubits stored
as the x_{N-1} = 0 half, the top qubit's RX as one mirror pass per level.

The reference's states are exactly flip-symmetric (psi(x) == psi(~x) bit for
bit), so the exact schedule on the half must reproduce the reference bit for
bit once mirrored; the fast schedule stays within the north star's 1e-12."""

import hashlib

import numpy as np
import pytest

import paper_2312_03019_b200 as Q

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("n,betas", [
    (13, (0.4, 1.1)),
    (16, (0.3, 2.9, 1.0)),        # second RX form on one level (fast mode)
    (21, (2.95, 3.05)),           # odd n: u3r(20) + an isolated node
    (24, (0.8, 2.2, 3.0, 0.1)),   # three local sets
])
def test_symmetric_matches_full_state(oracle, n, betas):
    g = Q.random_regular_graph(n, 3, seed=n) if n % 2 == 0 else \
        Q.Graph.from_edges(n, list(Q.random_regular_graph(n - 1, 3, seed=n).edges))
    gammas = tuple(0.2 + 0.9 * k for k in range(len(betas)))
    pr = Q.QaoaParams(gammas, betas)
    ref = oracle.simulate(n, g.row_mask, g.tot_edge, gammas, betas)
    assert np.array_equal(ref, ref[::-1])  # the reference's state is flip-symmetric bit for bit
    eref = oracle.expectation(n, g.row_mask, ref)
    ex = Q.simulate(g, pr, "bitwise", exact=True, symmetric=True, max_qubits=n)
    assert isinstance(ex, Q.SymmetricState)
    assert ex.expectation(g) == pytest.approx(eref, rel=1e-10)
    assert ex.norm() == pytest.approx(1.0, abs=1e-12)
    assert np.array_equal(ex.amps, ref)
    fa = Q.simulate(g, pr, "bitwise", symmetric=True, max_qubits=n)
    assert Q.expectation(g, fa) == pytest.approx(eref, rel=1e-10)
    assert np.max(np.abs(fa.amps - ref)) <= 1e-12


def test_symmetric_golden_n26_sha(golden):
    """Config C2 (u3r N=26 p=4): the exact schedule on the 2^25 half, mirrored,
    has the SHA-256 of the reference's own full state."""
    meta, _ = golden
    b = next(x for x in meta["big"] if x["key"] == "u3r26_p4")
    g = Q.random_regular_graph(26, 3, seed=0)
    pr = Q.params_from_seed(4, 0)
    s = Q.simulate(g, pr, "bitwise", exact=True, symmetric=True, max_qubits=26)
    assert Q.expectation(g, s) == pytest.approx(b["expectation"], rel=1e-10)
    assert sha(s.amps) == b["amps_sha256"]


def test_symmetric_state_operations():
    """copy, max_abs_diff between halves, device materialisation (engine())
    followed by a single-qubit gate, reuse as state=."""
    n = 18
    g = Q.random_regular_graph(n, 3, seed=2)
    pr = Q.params_from_seed(3, 1)
    full = Q.simulate(g, pr, "bitwise", max_qubits=n)
    sym = Q.simulate(g, pr, "bitwise", symmetric=True, max_qubits=n)
    c = sym.copy()
    assert Q.max_abs_diff(sym, c) == 0.0
    assert Q.max_abs_diff(sym, full) <= 1e-12
    again = Q.simulate(g, pr, "bitwise", symmetric=True, max_qubits=n, state=c)
    assert again is c and Q.max_abs_diff(again, sym) == 0.0
    eng = sym.engine()  # full-size device copy
    assert eng.n == n and not isinstance(sym.half_engine, Q.Engine)
    Q.apply_rx(sym, 3, 0.7)
    Q.apply_rx(full, 3, 0.7)
    assert Q.max_abs_diff(sym, full) <= 1e-12
    with pytest.raises(ValueError):
        Q.simulate(g, pr, "bitwise", symmetric=True, launch_control=False, max_qubits=n)


def _free_gib():
    import torch

    return torch.cuda.mem_get_info(0)[0] / 2**30


def test_symmetric_n31_against_full():
    """N=31 (odd: u3r(30) + isolated node): the 16 GiB half against the 32 GiB
    full state, <C> and 64 sample blocks of 4096 amplitudes."""
    if _free_gib() < 60:
        pytest.skip("needs 60 GiB")
    n = 31
    g = Q.Graph.from_edges(n, list(Q.random_regular_graph(30, 3, seed=0).edges))
    pr = Q.params_from_seed(3, 0)
    offs = np.linspace(0, (1 << n) - 4096, 64).astype(np.int64) // 4096 * 4096
    full = Q.simulate(g, pr, "bitwise", max_qubits=n)
    e_full = Q.expectation(g, full)
    blocks_full = np.concatenate([full.engine().read(int(o), 4096) for o in offs])
    full.engine().close()
    sym = Q.simulate(g, pr, "bitwise", symmetric=True, max_qubits=n)
    h = 1 << (n - 1)
    he = sym.half_engine
    blocks = []
    for o in offs:
        o = int(o)
        if o < h:
            blocks.append(he.read(o, 4096))
        else:  # psi(x) = psi(~x): the mirrored block of the half, reversed
            lo = (1 << n) - 1 - (o + 4095)
            blocks.append(he.read(lo, 4096)[::-1])
    assert np.max(np.abs(np.concatenate(blocks) - blocks_full)) <= 1e-12
    assert Q.expectation(g, sym) == pytest.approx(e_full, rel=1e-10)
    he.close()


def test_symmetric_n34_p1_closed_form():
    """N=34 on ONE B200 (the half is 128 GiB; the full state would not fit):
    p=1 per-edge closed form and the norm."""
    if _free_gib() < 132:
        pytest.skip("needs 132 GiB")
    from oracle import oracle as O

    g = Q.random_regular_graph(34, 3, seed=0)
    gm, bt = O.params_from_seed(1, 0)
    s = Q.simulate(g, Q.QaoaParams(gm, bt), "bitwise", symmetric=True, max_qubits=34)
    try:
        assert Q.expectation(g, s) == pytest.approx(16.931923255348405, rel=1e-10)
        assert s.norm() == pytest.approx(1.0, abs=1e-12)
    finally:
        s.half_engine.close()


@pytest.mark.parametrize("n,betas", [
    (13, (0.4, 1.1, 2.0)),          # 12 local qubits: mirror low set + one 1-bit high set
    (17, (0.9, 2.8)),               # two sets: the mirror low set is merged / first / last
    (22, (0.3, 2.9, 1.0, 2.7)),     # second-form levels
    (23, (2.95, 0.2, 3.05, 1.4, 0.6)),  # odd: u3r(22) + isolated node; three sets
    (26, (0.7, 1.9, 2.6)),
])
def test_fused_mirror_matches_segmented_and_oracle(oracle, n, betas):
    """The mirror low set (local qubits 0..10 plus the virtual top qubit in one
    sweep, one qaoa_run_layers call) against the segmented run (one mirror pass
    per level) and the oracle's full state: amplitudes within 1e-12, <C> 1e-10."""
    from paper_2312_03019_b200.symmetric import simulate_symmetric

    g = Q.random_regular_graph(n, 3, seed=n) if n % 2 == 0 else \
        Q.Graph.from_edges(n, list(Q.random_regular_graph(n - 1, 3, seed=n).edges))
    gammas = tuple(0.3 + 0.7 * k for k in range(len(betas)))
    pr = Q.QaoaParams(gammas, betas)
    ref = oracle.simulate(n, g.row_mask, g.tot_edge, gammas, betas)
    eref = oracle.expectation(n, g.row_mask, ref)
    fu = simulate_symmetric(g, pr, fused=True)
    seg = simulate_symmetric(g, pr, fused=False)
    e_fu, e_seg = fu.expectation(g), seg.expectation(g)
    assert e_fu == pytest.approx(eref, rel=1e-10) and e_seg == pytest.approx(eref, rel=1e-10)
    a_fu, a_seg = fu.amps, seg.amps
    assert np.max(np.abs(a_fu - ref)) <= 1e-12
    assert np.max(np.abs(a_fu - a_seg)) <= 1e-13
    assert fu.norm() == pytest.approx(1.0, abs=1e-12)


def test_fused_mirror_refusals():
    """QAOA_RUN_MIRROR without QAOA_RUN_SHARDED: fast schedule and a graph of
    n_local + 1 nodes; anything else is refused with a message."""
    from paper_2312_03019_b200 import _lib
    from paper_2312_03019_b200.circuit import level_arrays
    from paper_2312_03019_b200.symmetric import simulate_symmetric

    pr = Q.params_from_seed(2, 0)
    g24 = Q.random_regular_graph(24, 3, seed=1)
    eng = Q.Engine(22)
    try:
        eng.ensure_graph(g24)  # 24 nodes on 22 local qubits: not a half state
        tables, cs, ss = level_arrays(g24, pr)
        with pytest.raises(ValueError, match="n_local \\+ 1"):
            eng.call("qaoa_run_layers", 2, _lib.dptr(np.ascontiguousarray(tables).view(np.float64)),
                     _lib.dptr(cs), _lib.dptr(ss), _lib.RUN_MIRROR)
    finally:
        eng.close()


@pytest.mark.parametrize("betas", [(0.4, 1.1, 2.0, 0.7), (2.9, 0.3, 2.2)])
def test_fused_mirror_swapped_layout_bit_identical(betas):
    """Mirror low-set sweeps written out of place into the swapped qubit layout
    (high sets 11..15 and 16..20 of a 21-qubit half exchanged) equal the in-place
    run bit for bit (N = 22)."""
    from paper_2312_03019_b200.symmetric import simulate_symmetric

    n = 22
    g = Q.random_regular_graph(n, 3, seed=5)
    pr = Q.QaoaParams(tuple(0.5 + 0.6 * k for k in range(len(betas))), betas)
    runs = []
    for mode in (0, 1):
        s = simulate_symmetric(g, pr)
        s.half_engine.call("qaoa_set_layout_swap", mode)
        s = simulate_symmetric(g, pr, state=s)
        runs.append((s.expectation(g), s.amps.copy()))
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])


@pytest.mark.parametrize("betas", [(2.9,), (2.9, 0.4), (0.3, 2.8, 3.0), (0.5, 1.0)])
def test_symmetric_expectation_only(betas):
    """store_state=False (the optimizer's evaluations): the last sweep only reads;
    <C> is right whatever the parity of second-form levels (which complement the
    virtual top bit) and the state refuses reads."""
    n = 20
    g = Q.random_regular_graph(n, 3, seed=7)
    pr = Q.QaoaParams(tuple(0.4 + 0.8 * k for k in range(len(betas))), betas)
    e_full = Q.expectation(g, Q.simulate(g, pr, "bitwise", max_qubits=n))
    s = Q.simulate(g, pr, "bitwise", symmetric=True, store_state=False, max_qubits=n)
    assert Q.expectation(g, s) == pytest.approx(e_full, rel=1e-10)
    with pytest.raises(Exception):
        s.amps


@pytest.mark.parametrize("n,betas", [(13, (0.4, 2.9)), (16, (1.1, 0.3, 2.2)), (21, (2.95, 0.6)),
                                     (25, (0.8, 2.7, 1.3))])
def test_exact_fold_matches_reference_order(oracle, n, betas):
    """Exact schedule in one call: the virtual top qubit folded into the top
    set (after that set's qubits) is bit for bit the reference -- and the
    segmented run with its separate mirror passes."""
    from paper_2312_03019_b200.symmetric import simulate_symmetric

    g = Q.random_regular_graph(n, 3, seed=n + 1) if n % 2 == 0 else \
        Q.Graph.from_edges(n, list(Q.random_regular_graph(n - 1, 3, seed=n).edges))
    pr = Q.QaoaParams(tuple(0.7 + 0.5 * k for k in range(len(betas))), betas)
    ref = oracle.simulate(n, g.row_mask, g.tot_edge, pr.gamma, pr.beta)
    fo = simulate_symmetric(g, pr, exact=True)
    seg = simulate_symmetric(g, pr, exact=True, fused=False)
    assert np.array_equal(fo.amps, ref)
    assert np.array_equal(seg.amps, ref)


@pytest.mark.parametrize("n,p", [(14, 2), (20, 3), (24, 2)])
def test_weighted_symmetric_matches_full(n, p):
    """Weighted graphs (compressed backend, factored weighted cost): the mirror
    low set with the weighted cut basis against the full-state fast run
    (amplitudes 1e-12, weighted <C> 1e-10), fused and read-back <C>."""
    g = Q.random_regular_graph(n, 3, weighted=True, seed=n)
    assert not g.is_unweighted
    pr = Q.params_from_seed(p, n)
    full = Q.simulate(g, pr, "compressed", max_qubits=n)
    e_full = Q.expectation(g, full)
    a_full = full.amps
    sym = Q.simulate(g, pr, "compressed", symmetric=True, max_qubits=n)
    assert isinstance(sym, Q.SymmetricState)
    assert Q.expectation(g, sym) == pytest.approx(e_full, rel=1e-10)
    assert np.max(np.abs(sym.amps - a_full)) <= 1e-12
    # unfused <C> of a weighted half state (read-only reduction, doubled)
    s2 = Q.simulate(g, pr, "compressed", symmetric=True, max_qubits=n, fuse_expectation=False)
    assert Q.expectation(g, s2) == pytest.approx(e_full, rel=1e-10)
    with pytest.raises(ValueError):
        Q.simulate(g, pr, "compressed", symmetric=True, exact=True, max_qubits=n)


def test_symmetric_sampling_in_place():
    """Sampling a symmetric half state walks the virtual full index space on the
    device (qaoa_set_mirror): the same draws as sampling the full state, and no
    full-size copy is made."""
    n = 20
    g = Q.random_regular_graph(n, 3, seed=9)
    pr = Q.params_from_seed(3, 2)
    full = Q.simulate(g, pr, "bitwise", exact=True, max_qubits=n)
    sym = Q.simulate(g, pr, "bitwise", exact=True, symmetric=True, max_qubits=n)
    a = Q.sample(full, 4000, seed=5)
    b = Q.sample(sym, 4000, seed=5)
    assert sym.half_engine is not None  # still the half: nothing materialised
    assert np.array_equal(a, b)
    assert b.min() >= 0 and b.max() < (1 << n)
    assert (b >= (1 << (n - 1))).any()  # draws from the mirrored half too
