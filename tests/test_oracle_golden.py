"""Pin the CPU oracle (oracle/qaoa_oracle.c) to the reference's own outputs.

The golden fixtures were produced by running the reference package
(tests/golden/make_golden.py); the oracle must reproduce them bit for bit
(amplitudes, cut tables) and within 1e-10 relative for <C> (numpy's pairwise
sum cannot be bit-matched).  Only after this does the oracle check the GPU.
"""

import hashlib
import math

import numpy as np
import pytest


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def masks_of(n, edges):
    m = [0] * n
    for i, j in edges:
        m[min(i, j)] |= 1 << max(i, j)
    return m


def test_small_cases_bit_exact(golden, oracle):
    meta, arrays = golden
    for case in meta["cases"]:
        n = case["n"]
        rm = masks_of(n, case["edges"])
        amps = oracle.simulate(n, rm, case["tot_edge"], case["gamma"], case["beta"], threads=1)
        assert np.array_equal(amps, arrays["amps_" + case["name"]]), case["name"]
        cut = oracle.cut_counts(n, rm)
        assert np.array_equal(cut, arrays["cut_" + case["name"]]), case["name"]
        e = oracle.expectation(n, rm, amps)
        assert e == pytest.approx(case["expectation"], rel=1e-12, abs=1e-12)


def test_single_layers_bit_exact(golden, oracle):
    meta, arrays = golden
    L = meta["layer"]
    rm = masks_of(L["n"], L["edges"])
    a = arrays["layer_in"].copy()
    oracle.apply_cost(a, L["n"], rm, len(L["edges"]), L["gamma"])
    assert np.array_equal(a, arrays["layer_cost_out"])
    oracle.apply_mixer(a, L["n"], L["beta"])
    assert np.array_equal(a, arrays["layer_mix_out"])


@pytest.mark.parametrize("key", ["u3r16_p2", "u3r18_p4", "u3r20_p1", "u3r20_p3"])
def test_larger_cases_hash(golden, oracle, key):
    meta, arrays = golden
    b = next(x for x in meta["big"] if x["key"] == key)
    edges = meta["graphs"].get(f"u3r{b['n']}_seed0")
    if edges is None:
        edges = oracle.random_regular_edges(b["n"], 3, 0)
    rm = masks_of(b["n"], edges)
    gm, bt = oracle.params_from_seed(b["p"], 0)
    amps = oracle.simulate(b["n"], rm, len(edges), gm, bt)
    assert sha(amps) == b["amps_sha256"]
    assert sha(oracle.cut_counts(b["n"], rm)) == b["cut_sha256"]
    assert oracle.expectation(b["n"], rm, amps) == pytest.approx(b["expectation"], rel=1e-10)


def test_generators_match_reference(golden, oracle):
    meta, _ = golden
    for key, edges in meta["graphs"].items():
        if not key.startswith("u3r"):
            continue
        n = int(key[3:].split("_")[0])
        seed = int(key.split("seed")[1])
        assert [list(e) for e in oracle.random_regular_edges(n, 3, seed)] == edges, key
    for key, pr in meta["params"].items():
        p = int(key[1:].split("_")[0])
        gm, bt = oracle.params_from_seed(p, 0)
        assert list(gm) == pr["gamma"] and list(bt) == pr["beta"]


def test_phase_table_expression(golden, oracle):
    meta, arrays = golden
    tab = oracle.phase_table(3, 0.9)
    assert [[float(v.real), float(v.imag)] for v in tab] == meta["kat"]["phase_table_E3_g0.9"]
    assert np.array_equal(oracle.phase_table(45, 4.002148315014479), arrays["phase_table_E45"])


def test_p1_closed_form_matches_oracle(golden, oracle):
    # the per-edge closed form reproduces the reference at p=1
    meta, _ = golden
    b = next(x for x in meta["big"] if x["key"] == "u3r20_p1")
    edges = [tuple(e) for e in meta["graphs"]["u3r20_seed0"]]
    gm, bt = oracle.params_from_seed(1, 0)
    cf = oracle.p1_closed_form(20, edges, gm[0], bt[0])
    assert cf == pytest.approx(b["expectation"], rel=1e-12)


def test_oracle_invariants(oracle):
    n = 12
    edges = oracle.random_regular_edges(n, 3, 5)
    rm = oracle.row_masks(n, edges)
    cut = oracle.cut_counts(n, rm)
    assert cut.sum() == len(edges) * (1 << (n - 1))       # sum_x C(x) = E 2^(n-1)
    assert np.array_equal(cut, cut[::-1])                  # C(x) = C(~x)
    gm, bt = oracle.params_from_seed(3, 1)
    amps = oracle.simulate(n, rm, len(edges), gm, bt)
    assert oracle.norm(n, amps) == pytest.approx(1.0, abs=1e-13)


# ---- gate-level path (backend "baseline", launch_control=False) -------------
def _gates_golden():
    import json
    import os

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    with open(os.path.join(here, "golden_gates.json")) as f:
        meta = json.load(f)
    return meta, dict(np.load(os.path.join(here, "golden_gates.npz")))


def test_oracle_gate_level_circuits_bit_exact(oracle):
    """oracle.simulate_gates == the reference's simulate(backend="baseline"),
    with and without launch control, unweighted and weighted (fixtures made by
    running the reference, tests/golden/make_golden_gates.py)."""
    meta, arrays = _gates_golden()
    for case in meta["cases"]:
        got = oracle.simulate_gates(case["n"], case["edges"], case["gamma"], case["beta"],
                                    launch_control=case["launch_control"])
        assert np.array_equal(got, arrays["amps_" + case["name"]]), case["name"]


def test_oracle_single_gates_bit_exact(oracle):
    meta, arrays = _gates_golden()
    n = meta["gate_n"]
    a = arrays["gate_in"].copy()
    for k, op in enumerate(meta["gates"]):
        if op[0] == "h":
            oracle.apply_h(a, n, op[1])
        else:
            oracle.apply_rzz(a, n, op[1], op[2], op[3])
        assert np.array_equal(a, arrays[f"gate_out_{k}"]), op


def test_reference_states_are_flip_symmetric(golden):
    """The premise of the symmetric half-state mode, pinned on the REFERENCE's
    own outputs: every launch-control state it produced satisfies
    psi(x) == psi(~x) bit for bit (golden_small.npz, made by running it)."""
    meta, arrays = golden
    checked = 0
    for case in meta["cases"]:
        a = arrays["amps_" + case["name"]]
        assert np.array_equal(a, a[::-1]), case["name"]
        checked += 1
    assert checked >= 20
