"""Host-side logic of the drop-in API that needs no GPU: graph model and
generators (vs the reference's outputs), parameter / backend validation, the
memory guard, phase tables and the scalar bitwise primitives (the reference's
KATs, test_cost.py:63-75, test_acceptance.py:102-107)."""

import math

import numpy as np
import pytest

import paper_2312_03019_b200 as Q
from paper_2312_03019_b200 import cost, graph


def test_graph_generators_match_reference(golden):
    meta, _ = golden
    for key, edges in meta["graphs"].items():
        if key.startswith("u3r"):
            n = int(key[3:].split("_")[0])
            seed = int(key.split("seed")[1])
            g = Q.random_regular_graph(n, 3, seed=seed)
        else:
            n = int(key[2:].split("_")[0])
            g = Q.erdos_renyi_graph(n, 0.5, seed=0)
        assert [[i, j] for i, j, _ in g.edges] == edges, key
    assert Q.erdos_renyi_graph(33, 0.5, 0).tot_edge == 236


def test_graph_model():
    g = Q.Graph.from_edges(4, [(2, 1, 1.0), (0, 3, 1.0), (0, 1, 1.0)])
    assert g.edges == ((0, 1, 1.0), (0, 3, 1.0), (1, 2, 1.0))
    assert g.row_mask == (0b1010, 0b0100, 0, 0)
    assert g.tot_edge == 3 and g.is_unweighted
    assert sum(bin(m).count("1") for m in g.row_mask) == g.tot_edge
    with pytest.raises(ValueError):
        Q.Graph.from_edges(3, [(1, 1, 1.0)])
    with pytest.raises(ValueError):
        Q.Graph.from_edges(3, [(0, 1, 1.0), (1, 0, 1.0)])
    with pytest.raises(ValueError):
        Q.Graph.from_edges(65, [])
    with pytest.raises(ValueError):
        Q.Graph.from_edges(3, [(0, 5, 1.0)])
    assert not Q.Graph.from_edges(2, [(0, 1, 0.5)]).is_unweighted


def test_edge_list_roundtrip():
    g = Q.random_regular_graph(10, 3, seed=2)
    assert Q.parse_edge_list(Q.format_edge_list(g)) == g
    gw = Q.parse_edge_list("# c\n0 1 0.5\n1 2\n")
    assert gw.edges == ((0, 1, 0.5), (1, 2, 1.0))
    for bad in ("", "0 0", "0 1\n1 0", "0 x", "-1 2", "0 1 2 3"):
        with pytest.raises(graph.GraphParseError):
            Q.parse_edge_list(bad)


def test_generators_errors():
    with pytest.raises(ValueError):
        Q.random_regular_graph(5, 3)
    with pytest.raises(ValueError):
        Q.random_regular_graph(3, 3)
    with pytest.raises(ValueError):
        Q.cycle_graph(2)
    assert Q.complete_graph(6).tot_edge == 15
    assert Q.cycle_graph(9).tot_edge == 9


def test_params_and_backend_validation():
    with pytest.raises(ValueError):
        Q.QaoaParams(gamma=(0.1,), beta=(0.1, 0.2))
    with pytest.raises(ValueError):
        Q.QaoaParams(gamma=(), beta=())
    assert Q.QaoaParams(gamma=(1, 2), beta=(3, 4)).p == 2
    with pytest.raises(ValueError, match="unknown backend"):
        Q.validate_backend("fast")
    gw = Q.random_regular_graph(6, 3, weighted=True, seed=0)
    with pytest.raises(ValueError, match="unweighted"):
        Q.validate_backend("bitwise", gw)


def test_qubit_budget_guard():
    with pytest.raises(ValueError, match="GiB"):
        Q.check_qubit_budget(40)
    with pytest.raises(ValueError):
        Q.check_qubit_budget(0)
    Q.check_qubit_budget(30, max_qubits=30)
    g = Q.random_regular_graph(28, 3, seed=0)
    with pytest.raises(ValueError, match="GiB"):  # raised before any device work
        Q.simulate(g, Q.QaoaParams((0.1,), (0.2,)), "bitwise")


def test_phase_table_and_rx_coefficients(golden):
    meta, arrays = golden
    assert [[float(v.real), float(v.imag)] for v in Q.phase_table(3, 0.9)] == \
        meta["kat"]["phase_table_E3_g0.9"]
    assert np.array_equal(Q.phase_table(45, 4.002148315014479), arrays["phase_table_E45"])
    c, s = Q.rx_coefficients(0.8)
    assert c == math.cos(-0.4) and s == math.sin(-0.4)


def test_bitwise_primitives(golden):
    meta, _ = golden
    assert list(cost.row_cut_count(0b00010110, 0b00001011, 1, word_bits=8)) == meta["kat"]["row_step"]
    assert cost.broadcast_bit(0b100, 2, word_bits=8) == 0xFF
    assert cost.broadcast_bit(0b011, 2, word_bits=8) == 0
    tri = Q.Graph.from_edges(3, [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0)])
    plan = Q.CompressedCostPlan(tri)
    assert Q.cut_edge_count_bitwise(plan, 0b011) == 2
    assert Q.total_rotation_unweighted(plan, 0b011) == -1
    sq = Q.Graph.from_edges(4, [(0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0), (0, 3, 1.0)])
    assert Q.total_rotation_unweighted(Q.CompressedCostPlan(sq), 0b0101) == -4
    g = Q.random_regular_graph(10, 3, seed=1)
    p = Q.CompressedCostPlan(g)
    for b in range(0, 1 << 10, 37):
        assert Q.total_rotation_unweighted(p, b) == Q.total_rotation_weighted(p, b)
        assert Q.cut_edge_count_bitwise(p, b) == int(Q.cut_value(g, b))


def test_gate_counts():
    g = Q.complete_graph(30)
    h, rzz, rx = Q.gate_counts(30, g, 1)
    assert (h, rzz, rx) == (30, 435, 30)
    assert rzz / (h + rzz + rx) == pytest.approx(0.879, abs=1e-3)


def test_level_arrays_shape():
    g = Q.random_regular_graph(8, 3, seed=0)
    pr = Q.QaoaParams((0.3, 0.4), (0.5, 0.6))
    t, cs, ss = Q.level_arrays(g, pr)
    assert t.shape == (2, 2 * g.tot_edge + 1) and t.dtype == np.complex128
    assert cs[1] == math.cos(-0.3) and ss[0] == math.sin(-0.25)


def test_params_from_seed_matches_reference(golden):
    meta, _ = golden
    for key, pr in meta["params"].items():
        p = int(key[1:].split("_")[0])
        q = Q.params_from_seed(p, 0)
        assert list(q.gamma) == pr["gamma"] and list(q.beta) == pr["beta"]


def test_linear_ramp_and_wrap():
    from paper_2312_03019_b200.optimize import wrap_angles

    pr = Q.linear_ramp_params(4)
    assert pr.gamma[0] == pytest.approx(0.125 * math.pi / 2) and pr.beta[-1] == pytest.approx(0.125 * math.pi / 2)
    w = wrap_angles(np.array([7.0, -1.0, 4.0, -0.5]), 2)
    assert 0 <= w.gamma[0] < 2 * math.pi and 0 <= w.beta[1] < math.pi
