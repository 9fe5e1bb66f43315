"""The drop-in API on the GPU, mirroring the reference's own tests
(pkg/tests/test_circuit.py, test_state.py, test_acceptance.py criteria 4/6)."""

import math

import numpy as np
import pytest

import paper_2312_03019_b200 as Q

pytestmark = pytest.mark.gpu

TRIANGLE = Q.Graph.from_edges(3, [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0)])
SINGLE_EDGE = Q.Graph.from_edges(2, [(0, 1, 1.0)])


def test_init_uniform_values():
    np.testing.assert_array_equal(Q.init_uniform(2).amps, np.full(4, 0.5))
    np.testing.assert_allclose(Q.init_uniform(3).amps, np.full(8, 1 / (2 * math.sqrt(2))))
    assert Q.init_uniform(20).amps[12345] == math.sqrt(1.0 / (1 << 20))
    with pytest.raises(ValueError, match="GiB"):
        Q.init_uniform(40)


def test_zero_angles_identity():
    g = Q.random_regular_graph(6, 3, seed=0)
    s = Q.simulate(g, Q.QaoaParams((0.0,), (0.0,)), "bitwise")
    assert Q.max_abs_diff(s, Q.init_uniform(6)) < 1e-14


def test_single_edge_closed_form():
    for gamma in np.linspace(0.0, 2.0 * math.pi, 8, endpoint=False):
        for beta in np.linspace(0.0, math.pi, 8, endpoint=False):
            s = Q.simulate(SINGLE_EDGE, Q.QaoaParams((float(gamma),), (float(beta),)), "bitwise")
            closed = 0.5 * (1.0 + math.sin(2.0 * beta) * math.sin(gamma))
            assert abs(Q.expectation(SINGLE_EDGE, s) - closed) <= 1e-12


def test_single_edge_closed_form_embedded_grid():
    # one edge inside a 14-node graph: the other 12 isolated nodes exercise the tiled path
    g = Q.Graph.from_edges(14, [(5, 9, 1.0)])
    for gamma, beta in ((0.3, 0.2), (2.0, 1.0), (4.0, 2.9)):
        s = Q.simulate(g, Q.QaoaParams((gamma,), (beta,)), "bitwise")
        closed = 0.5 * (1.0 + math.sin(2.0 * beta) * math.sin(gamma))
        assert Q.expectation(g, s) == pytest.approx(closed, abs=1e-12)


def test_expectation_kats():
    assert Q.expectation(TRIANGLE, Q.init_uniform(3)) == pytest.approx(1.5)
    amps = np.zeros(4, dtype=np.complex128)
    amps[0b01] = 1.0
    assert Q.expectation(SINGLE_EDGE, Q.StateVector(2, amps)) == 1
    g = Q.random_regular_graph(6, 3, seed=1)
    amps = np.zeros(64, dtype=np.complex128)
    amps[0] = 1.0
    assert Q.expectation(g, Q.StateVector(6, amps)) == 0
    with pytest.raises(ValueError):
        Q.expectation(TRIANGLE, Q.init_uniform(4))


def test_backends_and_knobs_identical():
    g = Q.random_regular_graph(8, 3, seed=5)
    pr = Q.QaoaParams((0.4, 1.7), (0.8, 2.5))
    plain = Q.simulate(g, pr, "bitwise")
    for kw in ({"backend": "compressed"}, {"threads": 3}, {"batch_width": 4}):
        kw = {"backend": "bitwise", **kw}
        other = Q.simulate(g, pr, **kw)
        assert Q.max_abs_diff(plain, other) == 0
    # the gate-level backend and the Hadamard-chain init round differently
    # (the reference's own 1e-10 equivalence gate, bench.py:16)
    for kw in ({"backend": "baseline"}, {"launch_control": False},
               {"backend": "baseline", "launch_control": False}):
        kw = {"backend": "bitwise", **kw}
        assert Q.max_abs_diff(plain, Q.simulate(g, pr, **kw)) <= 1e-12
    with pytest.raises(ValueError):
        Q.simulate(g, pr, "bitwise", batch_width=3)


def test_errors():
    with pytest.raises(ValueError, match="unknown backend"):
        Q.simulate(TRIANGLE, Q.QaoaParams((0.1,), (0.1,)), "fast")
    gw = Q.random_regular_graph(6, 3, weighted=True, seed=0)
    with pytest.raises(ValueError, match="unweighted"):
        Q.simulate(gw, Q.QaoaParams((0.1,), (0.1,)), "bitwise")
    s = Q.init_uniform(4)
    with pytest.raises(IndexError):
        Q.apply_rx(s, 4, 0.3)
    with pytest.raises(ValueError, match="qubits but graph"):
        Q.apply_cost_layer(s, TRIANGLE, 0.3, "bitwise")


def test_norm_preservation():
    for seed in range(5):
        rng = np.random.default_rng(seed)
        n = 14
        a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        a /= np.linalg.norm(a)
        s = Q.StateVector(n, a)
        Q.apply_mixer_layer(s, rng.uniform(0, math.pi))
        Q.apply_rx(s, 5, rng.uniform(0, math.pi))
        assert s.norm() == pytest.approx(1.0, abs=1e-12)


def test_rx_kats():
    # RX(pi) on |0> = -i|1>  (reference test_state.py RX KAT family)
    amps = np.zeros(2, dtype=np.complex128)
    amps[0] = 1.0
    s = Q.StateVector(1, amps)
    Q.apply_rx(s, 0, math.pi)
    np.testing.assert_allclose(s.amps, [0, -1j], atol=1e-15)


def test_host_roundtrip_and_copy():
    rng = np.random.default_rng(3)
    a = rng.normal(size=1 << 15) + 1j * rng.normal(size=1 << 15)
    s = Q.StateVector(15, a.copy())
    s.engine()                      # upload
    assert np.array_equal(s.amps, a)
    s.amps[7] = 2.0                 # host copy is authoritative after .amps
    assert s.engine().read(7, 1)[0] == 2.0
    c = s.copy()
    assert Q.max_abs_diff(s, c) == 0


def test_permutation_equivariance():
    rng = np.random.default_rng(11)
    for trial in range(4):
        n = 14
        g = Q.random_regular_graph(n, 3, seed=trial)
        perm = rng.permutation(n)
        rel = Q.Graph.from_edges(n, [(int(perm[i]), int(perm[j]), w) for i, j, w in g.edges])
        pr = Q.QaoaParams((0.5, 1.3), (0.7, 2.2))
        assert Q.expectation(g, Q.simulate(g, pr, "bitwise")) == pytest.approx(
            Q.expectation(rel, Q.simulate(rel, pr, "bitwise")), abs=1e-9)


def test_brute_force_uses_gpu_cut_table():
    g = Q.random_regular_graph(16, 3, seed=4)
    cut = Q.brute_force_max_cut(g)
    assert cut.value == max(Q.cut_value(g, b) for b in range(0, 1 << 16, 1))


def test_expectation_only_run():
    """store_state=False: the last sweep only reads; <C> is the stored run's, the
    state refuses amplitude reads and is reusable as a buffer (the optimizer's
    inner loop)."""
    g = Q.random_regular_graph(20, 3, seed=3)
    pr = Q.params_from_seed(3, 1)
    full = Q.simulate(g, pr, "bitwise")
    e_full = Q.expectation(g, full)
    for exact in (False, True):
        s = Q.simulate(g, pr, "bitwise", store_state=False, exact=exact)
        assert Q.expectation(g, s) == pytest.approx(e_full, rel=1e-10)
        with pytest.raises(Exception, match="not stored"):
            _ = s.amps
        s2 = Q.simulate(g, pr, "bitwise", state=s, exact=exact)
        assert np.max(np.abs(s2.amps - full.amps)) <= 1e-12


def test_new_entry_points_reject_bad_arguments():
    """The segmented-run, exchange and weighted entry points fail with the
    reference's exception types instead of launching."""
    import ctypes

    from paper_2312_03019_b200 import _lib

    L = _lib.load()
    g = Q.random_regular_graph(14, 3, seed=1)
    eng = Q.Engine(14)
    try:
        eng.ensure_graph(g)
        tables, cs, ss = Q.level_arrays(g, Q.params_from_seed(2, 0))
        t = np.ascontiguousarray(tables)
        nseg = ctypes.c_int()
        with pytest.raises(RuntimeError):  # no planned run yet
            eng.call("qaoa_run_segment", 0)
        eng.call("qaoa_run_begin", 2, _lib.dptr(t.view(np.float64)), _lib.dptr(cs), _lib.dptr(ss),
                 _lib.RUN_SHARDED, ctypes.byref(nseg))
        assert nseg.value >= 2
        with pytest.raises(IndexError):
            eng.call("qaoa_run_segment", nseg.value)
        with pytest.raises(IndexError):
            eng.call("qaoa_run_sweep_range", 0, 0, 10 ** 6)
        for k in range(nseg.value):
            eng.call("qaoa_run_segment", k)
        eng.call("qaoa_run_end")
        with pytest.raises(RuntimeError):  # weights not set
            eng.call("qaoa_run_layers_weighted", 1, _lib.dptr(np.array([0.3])), _lib.dptr(cs[:1]),
                     _lib.dptr(ss[:1]), 0)
        ptrs = (ctypes.c_void_p * 2)(eng.state_ptr(), eng.state_ptr())
        with pytest.raises(ValueError):  # g = 5 > 4
            _lib.check(L.qaoa_exchange(0, None, 5, ptrs, 14, 0, 0, 1, _lib.dptr(np.zeros(3)),
                                       _lib.dptr(np.array([1.0, 0.0]))))
        with pytest.raises(IndexError):  # swapped bits beyond the local qubits
            _lib.check(L.qaoa_exchange(0, None, 1, ptrs, 14, 14, 0, 1, _lib.dptr(np.zeros(3)),
                                       _lib.dptr(np.array([1.0, 0.0]))))
    finally:
        eng.close()


def test_plan_export_matches_engine_launch_count():
    """qaoa_plan (device-free) is the plan the engine runs: same sweep count (the
    engine's launch count adds the two launch-control helpers, basis_table_kernel
    and gen_table_kernel)."""
    import ctypes

    from paper_2312_03019_b200 import _lib

    g = Q.random_regular_graph(30, 3, seed=0)
    eng = Q.Engine(30)
    try:
        eng.ensure_graph(g)
        tables, cs, ss = Q.level_arrays(g, Q.params_from_seed(10, 0))
        t = np.ascontiguousarray(tables)
        eng.call("qaoa_run_layers", 10, _lib.dptr(t.view(np.float64)), _lib.dptr(cs), _lib.dptr(ss), 0)
        nl, hb = ctypes.c_int(), ctypes.c_double()
        _lib.load().qaoa_last_run_stats(eng.ptr, ctypes.byref(nl), ctypes.byref(hb))
        assert _lib.load().qaoa_plan(30, 10, 0, None, 0) == 21
        assert nl.value == 21 + 2
    finally:
        eng.close()


def test_pack_unpack_chunks_roundtrip():
    """qaoa_pack_chunks gathers chunk d (local bits L spelling d) in order of the
    remaining bits; unpack scatters back: a round trip is the identity and
    the packed order matches the definition."""
    import ctypes

    import torch

    n, g = 12, 2
    rng = np.random.default_rng(0)
    amps = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    s = Q.StateVector(n, amps.copy())
    eng = s.engine()
    bits = (ctypes.c_int * g)(3, 7)
    buf = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
    eng.call("qaoa_pack_chunks", g, bits, ctypes.c_void_p(buf.data_ptr()))
    packed = buf.cpu().numpy()
    idx = np.arange(1 << n)
    d = ((idx >> 3) & 1) | (((idx >> 7) & 1) << 1)
    expect = np.concatenate([amps[d == c] for c in range(1 << g)])
    assert np.array_equal(packed, expect)
    eng.call("qaoa_init_uniform")
    eng.call("qaoa_unpack_chunks", g, bits, ctypes.c_void_p(buf.data_ptr()))
    torch.cuda.synchronize()
    s._where = "device"
    assert np.array_equal(s.amps, amps)


def test_weighted_fused_regrow_tables_on_one_state():
    """Fused weighted runs with growing p on one reused state (the per-level
    tile tables grow; the <C> table must survive the regrow): p=1, then p=3,
    then p=2 each equal a fresh context's run (regression: a freed <C> table
    pointer was reused after the per-level tables grew)."""
    g = Q.random_regular_graph(16, 3, seed=4, weighted=True)
    s = None
    for gm, bt in (((0.7,), (0.4,)), ((0.3, 1.9, 0.8), (0.2, 2.7, 1.1)), ((1.2, 0.5), (0.9, 0.3))):
        pr = Q.QaoaParams(gm, bt)
        s = Q.simulate(g, pr, "compressed", state=s)
        e = Q.expectation(g, s)
        fresh = Q.simulate(g, pr, "compressed")
        assert Q.max_abs_diff(s, fresh) == 0.0
        assert e == Q.expectation(g, fresh)
