"""The gate-level path on the GPU: the reference's default backend "baseline"
(one RZZ pass per edge, one RX pass per qubit: circuit.py:76-80, 108-113,
state.py:110-149), init_state(launch_control=False) (|0..0> plus n Hadamards,
circuit.py:57-62, state.py:66-107), the single gates, and the per-index edge
sums rotation_totals (cost.py:77-86) / cut_values_array (graph.py:144-151).
Everything bit-identical to the reference (golden fixtures made by running it,
tests/golden/make_golden_gates.py) and to the oracle at larger sizes."""

import json
import os

import numpy as np
import pytest

import paper_2312_03019_b200 as Q

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def gates_golden():
    with open(os.path.join(HERE, "golden_gates.json")) as f:
        meta = json.load(f)
    return meta, dict(np.load(os.path.join(HERE, "golden_gates.npz")))


def _graph(case):
    return Q.Graph.from_edges(case["n"], [tuple(e) for e in case["edges"]])


def test_baseline_backend_golden(gates_golden):
    meta, arrays = gates_golden
    for case in meta["cases"]:
        g = _graph(case)
        pr = Q.QaoaParams(tuple(case["gamma"]), tuple(case["beta"]))
        Q.write_counter.reset()
        s = Q.simulate(g, pr, "baseline", launch_control=case["launch_control"], max_qubits=16)
        assert Q.write_counter.amp_writes == case["amp_writes"], case["name"]
        assert np.array_equal(s.amps, arrays["amps_" + case["name"]]), case["name"]
        assert Q.expectation(g, s) == pytest.approx(case["expectation"], rel=1e-10, abs=1e-12)


def test_init_state_without_launch_control_golden(gates_golden):
    meta, arrays = gates_golden
    for rec in meta["init"]:
        n = rec["n"]
        Q.write_counter.reset()
        s = Q.init_state(n, launch_control=False, max_qubits=16)
        assert Q.write_counter.amp_writes == rec["amp_writes"]
        assert np.array_equal(s.amps, arrays[f"init_nolc_{n}"])


def test_single_gates_golden(gates_golden):
    meta, arrays = gates_golden
    n = meta["gate_n"]
    s = Q.StateVector(n, arrays["gate_in"].copy())
    for k, op in enumerate(meta["gates"]):
        if op[0] == "h":
            Q.apply_h(s, op[1])
        else:
            Q.apply_rzz(s, op[1], op[2], op[3])
        assert np.array_equal(s.amps, arrays[f"gate_out_{k}"]), op


def test_gate_errors():
    s = Q.init_uniform(4)
    with pytest.raises(ValueError, match="distinct"):
        Q.apply_rzz(s, 2, 2, 0.3)
    with pytest.raises(IndexError):
        Q.apply_rzz(s, 0, 4, 0.3)
    with pytest.raises(IndexError):
        Q.apply_h(s, -1)


@pytest.mark.parametrize("n,lc,weighted", [(16, True, False), (20, False, False), (18, True, True)])
def test_baseline_backend_vs_oracle(oracle, n, lc, weighted):
    g = Q.random_regular_graph(n, 3, weighted=weighted, seed=n)
    pr = Q.params_from_seed(2, n)
    ref = oracle.simulate_gates(n, g.edges, pr.gamma, pr.beta, launch_control=lc)
    s = Q.simulate(g, pr, "baseline", launch_control=lc, max_qubits=n)
    assert np.array_equal(s.amps, ref)


@pytest.mark.parametrize("n", [9, 14, 22])
def test_bitwise_without_launch_control(oracle, n):
    """launch_control=False on the fused engine: the Hadamard-chain state is the
    starting point (RUN_FROM_STATE); exact schedule bit-identical to the
    reference's order (H chain, then cost + mixer layers), fast within 1e-12."""
    g = Q.random_regular_graph(n, 3, seed=1) if n % 2 == 0 else Q.erdos_renyi_graph(n, 0.4, 1)
    pr = Q.params_from_seed(3, 1)
    ref = np.zeros(1 << n, dtype=np.complex128)
    ref[0] = 1.0
    for q in range(n):
        oracle.apply_h(ref, n, q)
    for gm, bt in zip(pr.gamma, pr.beta):
        oracle.apply_cost(ref, n, g.row_mask, g.tot_edge, gm)
        oracle.apply_mixer(ref, n, bt)
    Q.write_counter.reset()
    e = Q.simulate(g, pr, "bitwise", launch_control=False, exact=True, max_qubits=n)
    assert Q.write_counter.amp_writes == (1 << n) * ((n + 1) + pr.p * (n + 1))
    assert np.array_equal(e.amps, ref)
    f = Q.simulate(g, pr, "bitwise", launch_control=False, max_qubits=n)
    assert np.max(np.abs(f.amps - ref)) <= 1e-12
    assert Q.expectation(g, f) == pytest.approx(oracle.expectation(n, g.row_mask, ref), rel=1e-10)


def test_gates_on_complemented_state(oracle):
    """Gates applied to a fast-schedule state whose storage is complemented
    (second RX form) act on the true state."""
    n = 14
    g = Q.random_regular_graph(n, 3, seed=3)
    pr = Q.QaoaParams((0.7, 1.3), (2.9, 0.4))  # one second-form level: complemented storage
    s = Q.simulate(g, pr, "bitwise", max_qubits=n)
    from paper_2312_03019_b200 import _lib
    import ctypes

    m = ctypes.c_uint64()
    s.engine().call("qaoa_get_cmask", ctypes.byref(m))
    assert m.value != 0
    ref = s.engine().read()  # true order
    for op in (("h", 3), ("rzz", 2, 9, 0.6), ("h", 0), ("rzz", 13, 1, -1.7)):
        if op[0] == "h":
            Q.apply_h(s, op[1])
            oracle.apply_h(ref, n, op[1])
        else:
            Q.apply_rzz(s, op[1], op[2], op[3])
            oracle.apply_rzz(ref, n, op[1], op[2], op[3])
    assert np.array_equal(s.amps, ref)


def _edge_sums_numpy(g, kind):
    idx = np.arange(1 << g.n, dtype=np.uint64)
    out = np.zeros(1 << g.n, dtype=np.float64)
    for i, j, w in g.edges:
        diff = ((idx >> np.uint64(i)) ^ (idx >> np.uint64(j))) & np.uint64(1)
        out += w * (1.0 - 2.0 * diff.astype(np.float64)) if kind == 0 else w * diff.astype(np.float64)
    return out


@pytest.mark.parametrize("weighted", [False, True])
def test_rotation_totals_and_cut_values(weighted):
    """The reference's own expressions (cost.py:77-86, graph.py:144-151) restated
    in numpy: bit-identical float64 tables."""
    g = Q.random_regular_graph(14, 3, weighted=weighted, seed=8)
    assert np.array_equal(Q.plan_for(g).rotation_totals(), _edge_sums_numpy(g, 0))
    assert np.array_equal(Q.cut_values_array(g), _edge_sums_numpy(g, 1))
    if not weighted:
        assert np.array_equal(Q.cut_values_array(g), Q.plan_for(g).cut_counts().astype(np.float64))
