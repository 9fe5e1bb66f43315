"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle and
the reference's golden outputs.

Contract (BASELINE.json north_star): cut table bit-exact; amplitudes within
1e-12 absolute (complex128); <C> within 1e-10 relative.  The engine's exact
schedule (exact=True) is held to bit equality with the reference.
"""

import hashlib
import math

import numpy as np
import pytest

import paper_2312_03019_b200 as Q

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-12   # north-star amplitude tolerance (absolute)
EXP_RTOL = 1e-10  # north-star <C> tolerance (relative)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def graph_from(n, edges):
    return Q.Graph.from_edges(n, [(i, j, 1.0) for i, j in edges])


def test_golden_cases(golden):
    """26 reference runs (n = 2..12, KAT graphs, the acceptance-test family)."""
    meta, arrays = golden
    for case in meta["cases"]:
        g = graph_from(case["n"], case["edges"])
        pr = Q.QaoaParams(tuple(case["gamma"]), tuple(case["beta"]))
        ref = arrays["amps_" + case["name"]]
        s = Q.simulate(g, pr, "bitwise", exact=True)
        assert np.array_equal(s.amps, ref), case["name"]
        assert Q.expectation(g, s) == pytest.approx(case["expectation"], rel=EXP_RTOL, abs=1e-12)
        f = Q.simulate(g, pr, "bitwise")
        assert np.max(np.abs(f.amps - ref)) <= AMP_TOL, case["name"]
        assert Q.expectation(g, f) == pytest.approx(case["expectation"], rel=EXP_RTOL, abs=1e-12)
        assert np.array_equal(Q.plan_for(g).cut_counts(), arrays["cut_" + case["name"]])


@pytest.mark.parametrize("key", ["u3r16_p2", "u3r18_p4", "u3r20_p1", "u3r20_p3", "u3r22_p4",
                                 "u3r26_p4"])
def test_golden_large_bit_exact(golden, key):
    """Reference states up to N=26 p=4 (config C2): SHA-256 of the whole exact
    state equals the reference's; fast schedule within 1e-12 on a stride sample."""
    meta, arrays = golden
    b = next(x for x in meta["big"] if x["key"] == key)
    n, p = b["n"], b["p"]
    g = Q.random_regular_graph(n, 3, seed=0)
    gm = tuple(meta["params"].get(f"p{p}_seed0", {}).get("gamma", ())) or None
    from oracle import oracle as O
    gm, bt = O.params_from_seed(p, 0)
    pr = Q.QaoaParams(gm, bt)
    s = Q.simulate(g, pr, "bitwise", exact=True, max_qubits=n)
    amps = s.amps
    assert sha(amps) == b["amps_sha256"]
    assert Q.expectation(g, s) == pytest.approx(b["expectation"], rel=EXP_RTOL)
    f = Q.simulate(g, pr, "bitwise", max_qubits=n)
    assert Q.expectation(g, f) == pytest.approx(b["expectation"], rel=EXP_RTOL)
    sample = f.amps[::b["sample_stride"]]
    assert np.max(np.abs(sample - arrays["sample_" + key])) <= AMP_TOL
    assert np.max(np.abs(f.amps - amps)) <= AMP_TOL


@pytest.mark.parametrize("n", [1, 2, 3, 5, 9, 11, 12, 13, 14, 15, 16, 17, 19, 21, 22, 23])
def test_against_oracle_sizes(oracle, n):
    """Every size class of the planner: per-gate path (n < 12), single low set
    (12), two sets with carry 11..3 (13..21), three sets (22, 23)."""
    if n == 1:
        g = Q.Graph.from_edges(1, [])
    elif n < 4:
        g = Q.complete_graph(n)
    elif n % 2:
        g = Q.erdos_renyi_graph(n, 0.35, seed=n)
    else:
        g = Q.random_regular_graph(n, 3, seed=n)
    for p, seed in ((1, 1), (2, 2), (5, 3)):
        gm, bt = oracle.params_from_seed(p, seed + n)
        pr = Q.QaoaParams(gm, bt)
        ref = oracle.simulate(n, g.row_mask, g.tot_edge, gm, bt)
        eref = oracle.expectation(n, g.row_mask, ref)
        s = Q.simulate(g, pr, "bitwise", exact=True, max_qubits=30)
        assert np.array_equal(s.amps, ref), (n, p)
        f = Q.simulate(g, pr, "bitwise", max_qubits=30)
        assert np.max(np.abs(f.amps - ref)) <= AMP_TOL, (n, p)
        if g.tot_edge:
            assert Q.expectation(g, f) == pytest.approx(eref, rel=EXP_RTOL)
            assert Q.expectation(g, s) == pytest.approx(eref, rel=EXP_RTOL)


def test_rx_forms_and_complement(oracle):
    """beta near pi makes |sin| > |cos|: those levels run in the second factored
    form with the global-complement bookkeeping; odd and even counts."""
    n = 20
    g = Q.random_regular_graph(n, 3, seed=11)
    for betas in ((2.9,), (2.9, 3.05), (0.2, 2.8, 3.1), (3.14159, 0.0, 1.5707963267948966)):
        gms = tuple(0.3 + 0.7 * k for k in range(len(betas)))
        pr = Q.QaoaParams(gms, betas)
        ref = oracle.simulate(n, g.row_mask, g.tot_edge, gms, betas)
        f = Q.simulate(g, pr, "bitwise")
        assert np.max(np.abs(f.amps - ref)) <= AMP_TOL, betas
        assert Q.expectation(g, f) == pytest.approx(oracle.expectation(n, g.row_mask, ref),
                                                    rel=EXP_RTOL)


def test_dense_graph_uint16_cut_table(oracle):
    """E > 255 switches the device cut table to uint16 (ER(0.5) N=33 has E=236;
    complete graphs go beyond)."""
    for g in (Q.complete_graph(24), Q.erdos_renyi_graph(24, 0.97, seed=1)):
        ct = Q.build_cut_table(g)
        assert g.tot_edge > 255
        assert np.array_equal(ct, oracle.cut_counts(g.n, g.row_mask))
        gm, bt = oracle.params_from_seed(2, 4)
        ref = oracle.simulate(g.n, g.row_mask, g.tot_edge, gm, bt)
        f = Q.simulate(g, Q.QaoaParams(gm, bt), "bitwise", max_qubits=30)
        assert np.max(np.abs(f.amps - ref)) <= AMP_TOL


@pytest.mark.parametrize("n", [4, 10, 11, 12, 13, 20, 25])
def test_cut_table_bit_exact(oracle, n):
    g = Q.random_regular_graph(n, 3, seed=7) if n % 2 == 0 else Q.erdos_renyi_graph(n, 0.5, 7)
    assert np.array_equal(Q.build_cut_table(g), oracle.cut_counts(n, g.row_mask))


def _cut_counts_numpy(row_mask, xs):
    """C(x) = sum_i popcount(row_mask[i] & (bcast(x_i) ^ x)) (cost.py:55-63, 88-99)."""
    c = np.zeros(xs.size, dtype=np.int64)
    for i, m in enumerate(row_mask):
        b = np.uint64(0) - ((xs >> np.uint64(i)) & np.uint64(1))
        c += np.bitwise_count(np.uint64(m) & (b ^ xs)).astype(np.int64)
    return c


@pytest.mark.parametrize("n_nodes,dense", [(34, False), (40, True)])
def test_cut_table_wide_graph_fixed_high_bits(n_nodes, dense):
    """Graphs beyond 32 nodes (64-bit masks) on a 2^20 local index space with the
    high node bits fixed by x_hi (the table of one shard): uint8 and uint16."""
    from paper_2312_03019_b200 import _lib

    g = Q.erdos_renyi_graph(n_nodes, 0.5, seed=3) if dense else Q.random_regular_graph(n_nodes, 3, 5)
    nl = 20
    rng = np.random.default_rng(n_nodes)
    eng = Q.Engine(nl)
    try:
        for _ in range(2):
            x_hi = int(rng.integers(0, 1 << (n_nodes - nl))) << nl
            masks = np.array(g.row_mask, dtype=np.uint64)
            eng.call("qaoa_set_graph", n_nodes, masks.ctypes.data_as(_lib._u64p), g.tot_edge, x_hi)
            eng.call("qaoa_build_cut_table")
            out = np.empty(1 << nl, dtype=np.int64)
            eng.call("qaoa_read_cut_table", 0, out.size, out.ctypes.data_as(_lib._i64p))
            xs = np.uint64(x_hi) | np.arange(1 << nl, dtype=np.uint64)
            assert np.array_equal(out, _cut_counts_numpy(g.row_mask, xs))
    finally:
        eng.close()


def test_cut_table_invariants_large():
    """N=28 (256 Mi states): sum_x C(x) = E 2^(N-1), C(x) = C(~x), 0 <= C <= E."""
    g = Q.random_regular_graph(28, 3, seed=0)
    ct = Q.build_cut_table(g)
    assert int(ct.sum()) == g.tot_edge * (1 << 27)
    assert np.array_equal(ct, ct[::-1])
    assert ct.min() == 0 and ct.max() <= g.tot_edge


def test_single_layers_bit_exact(golden):
    meta, arrays = golden
    L = meta["layer"]
    g = graph_from(L["n"], L["edges"])
    s = Q.StateVector(L["n"], arrays["layer_in"].copy())
    Q.apply_cost_layer(s, g, L["gamma"], "bitwise")
    assert np.array_equal(s.amps, arrays["layer_cost_out"])
    Q.apply_mixer_layer(s, L["beta"])
    assert np.array_equal(s.amps, arrays["layer_mix_out"])


@pytest.mark.parametrize("n", [14, 21])
def test_layers_and_rx_vs_oracle(oracle, n):
    g = Q.random_regular_graph(n, 3, seed=3) if n % 2 == 0 else Q.erdos_renyi_graph(n, 0.3, 3)
    rng = np.random.default_rng(n)
    a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    a /= np.linalg.norm(a)
    s = Q.StateVector(n, a.copy())
    ref = a.copy()
    Q.apply_cost_layer(s, g, 1.3, "bitwise")
    oracle.apply_cost(ref, n, g.row_mask, g.tot_edge, 1.3)
    Q.apply_mixer_layer(s, 0.4)
    oracle.apply_mixer(ref, n, 0.4)
    for q in (0, 3, n - 1):
        Q.apply_rx(s, q, 0.77)
        oracle.apply_rx(ref, n, q, 0.77)
    assert np.array_equal(s.amps, ref)
    assert Q.expectation(g, s) == pytest.approx(oracle.expectation(n, g.row_mask, ref),
                                                rel=EXP_RTOL)


def test_fused_expectation_equals_standalone(oracle):
    g = Q.random_regular_graph(24, 3, seed=2)
    pr = Q.QaoaParams((0.4, 1.1, 2.0), (0.3, 2.9, 1.0))
    s = Q.simulate(g, pr, "bitwise", max_qubits=24)
    fused = Q.expectation(g, s)
    s2 = Q.simulate(g, pr, "bitwise", max_qubits=24, fuse_expectation=False)
    assert Q.expectation(g, s2) == pytest.approx(fused, rel=1e-13)
    assert Q.max_abs_diff(s, s2) == 0.0


def test_determinism():
    g = Q.random_regular_graph(22, 3, seed=9)
    pr = Q.QaoaParams((0.4, 1.1), (0.3, 2.2))
    a = Q.simulate(g, pr, "bitwise", max_qubits=22)
    b = Q.simulate(g, pr, "bitwise", max_qubits=22)
    assert Q.max_abs_diff(a, b) == 0.0
    assert Q.expectation(g, a) == Q.expectation(g, b)


# ---- beyond the CPU's reach: size-independent properties -------------------

def test_p1_closed_form_n30_n32():
    """p=1 per-edge closed form at N=30 and N=32."""
    from oracle import oracle as O
    gm, bt = O.params_from_seed(1, 0)
    for n, expected in ((30, 15.30350510591025), (32, 16.3237387796376)):
        g = Q.random_regular_graph(n, 3, seed=0)
        cf = O.p1_closed_form(n, [(i, j) for i, j, _ in g.edges], gm[0], bt[0])
        assert cf == pytest.approx(expected, rel=1e-12)
        s = Q.simulate(g, Q.QaoaParams(gm, bt), "bitwise", max_qubits=n)
        assert Q.expectation(g, s) == pytest.approx(cf, rel=EXP_RTOL)
        assert s.norm() == pytest.approx(1.0, abs=1e-12)
        del s


def test_config_c3_exact_vs_fast_n30():
    """Config C3 (u3r N=30, p=10): bit-exact schedule vs fast schedule on the
    device, amplitudes within 1e-12, <C> within 1e-10, norm 1."""
    from oracle import oracle as O
    g = Q.random_regular_graph(30, 3, seed=0)
    gm, bt = O.params_from_seed(10, 0)
    pr = Q.QaoaParams(gm, bt)
    e = Q.simulate(g, pr, "bitwise", exact=True, max_qubits=30)
    f = Q.simulate(g, pr, "bitwise", max_qubits=30)
    assert Q.max_abs_diff(e, f) <= AMP_TOL
    ee, ef = Q.expectation(g, e), Q.expectation(g, f)
    assert ef == pytest.approx(ee, rel=EXP_RTOL)
    assert 0.0 <= ef <= g.tot_edge
    assert f.norm() == pytest.approx(1.0, abs=1e-12)


def test_weighted_compressed_golden(golden):
    """Weighted graphs through the compressed backend (cost.py:147-159) vs the
    reference's own runs: totals are bit-identical, only the device sincos
    differs from glibc's by <= 2 ulp."""
    meta, arrays = golden
    for case in meta["weighted"]:
        g = Q.Graph.from_edges(case["n"], [tuple(e) for e in case["edges"]])
        assert not g.is_unweighted
        pr = Q.QaoaParams(tuple(case["gamma"]), tuple(case["beta"]))
        for backend in ("compressed", "baseline"):
            s = Q.simulate(g, pr, backend)
            assert np.max(np.abs(s.amps - arrays["wamps_" + case["name"]])) <= AMP_TOL, case["name"]
            assert Q.expectation(g, s) == pytest.approx(case["expectation"], rel=EXP_RTOL, abs=1e-12)
        with pytest.raises(ValueError, match="unweighted"):
            Q.simulate(g, pr, "bitwise")


def test_weighted_expectation_bounds():
    g = Q.random_regular_graph(8, 3, weighted=True, seed=2)
    for seed in range(10):
        rng = np.random.default_rng(seed)
        amps = rng.normal(size=256) + 1j * rng.normal(size=256)
        amps /= np.linalg.norm(amps)
        val = Q.expectation(g, Q.StateVector(8, amps))
        assert 0 <= val <= g.total_weight + 1e-12
        ref = float(np.sum(np.abs(amps) ** 2 * np.array([Q.cut_value(g, b) for b in range(256)])))
        assert val == pytest.approx(ref, rel=1e-12)


def test_weighted_larger_against_unweighted_limit():
    """All-ones weights through the weighted kernel equal the integer path."""
    g = Q.random_regular_graph(20, 3, seed=5)
    gw = Q.Graph.from_edges(20, [(i, j, 1.0 + 1e-300) for i, j, _ in g.edges])
    pr = Q.QaoaParams((0.7, 2.1), (0.4, 1.9))
    a = Q.simulate(g, pr, "bitwise", exact=True)
    # identical weights but flagged weighted: force the compressed weighted kernels
    s = Q.init_uniform(20)
    plan = Q.CompressedCostPlan(g)
    from paper_2312_03019_b200 import cost as C
    eng = s.engine()
    eng.ensure_graph(g)
    eng.ensure_weights(g)
    for gm, bt in zip(pr.gamma, pr.beta):
        eng.call("qaoa_apply_cost_weighted", gm)
        Q.apply_mixer_layer(s, bt)
    assert np.max(np.abs(s.amps - a.amps)) <= AMP_TOL
    assert eng.scalar("qaoa_expectation_weighted") == pytest.approx(Q.expectation(g, a), rel=1e-12)


@pytest.mark.parametrize("n,dense", [(12, False), (13, True), (16, False), (20, False), (21, True),
                                     (22, False), (26, False), (25, True)])
def test_weighted_fused_fast_matches_exact(n, dense):
    """The fast schedule's factored weighted cost (fused sweeps) against the
    reference-order weighted path (edge-order totals, bit-identical to the
    reference): amplitudes <= 1e-12, <C> <= 1e-10 relative, including levels
    that take the second RX form (complement bookkeeping)."""
    rng = np.random.default_rng(n)
    base = Q.erdos_renyi_graph(n, 0.5, seed=n) if dense else Q.random_regular_graph(n, 3, seed=n)
    g = Q.Graph.from_edges(n, [(i, j, float(rng.uniform(0.1, 2.0))) for i, j, _ in base.edges])
    assert not g.is_unweighted
    for betas in ((0.4, 1.1), (2.9, 0.3, 3.05)):
        gammas = tuple(0.3 + 0.8 * k for k in range(len(betas)))
        pr = Q.QaoaParams(gammas, betas)
        ref = Q.simulate(g, pr, "compressed", max_qubits=30, exact=True)
        ref_amps = ref.amps
        e_ref = Q.expectation(g, ref)
        f = Q.simulate(g, pr, "compressed", max_qubits=30)
        e_f = Q.expectation(g, f)  # fused into the last sweep
        assert np.max(np.abs(f.amps - ref_amps)) <= AMP_TOL, (n, betas)
        assert e_f == pytest.approx(e_ref, rel=EXP_RTOL)
        o = Q.simulate(g, pr, "compressed", max_qubits=30, store_state=False)
        assert Q.expectation(g, o) == pytest.approx(e_ref, rel=EXP_RTOL)
