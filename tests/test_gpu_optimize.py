"""Device-resident optimizer loop against the reference's
own Nelder-Mead traces (tests/golden/golden_optimize.json) and the reference's
optimizer acceptance criteria (test_acceptance.py criteria 6 and 10)."""

import json
import math
import os

import pytest

import paper_2312_03019_b200 as Q

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_optimize.json")


def test_traces_match_reference():
    for run in json.load(open(GOLDEN)):
        g = Q.random_regular_graph(run["n"], 3, seed=run["seed"])
        rep = Q.optimize(g, p=run["p"], backend="bitwise", budget=run["budget"], seed=run["seed"],
                         init_strategy=run["init"])
        ref = run["report"]
        assert rep.evaluations == ref["evaluations"]
        for (i, v), (ri, rv) in zip(rep.history, ref["history"]):
            assert i == ri and v == pytest.approx(rv, rel=1e-10)
        assert list(rep.best_params.gamma) == pytest.approx(ref["best_gamma"], abs=1e-12)
        assert list(rep.best_params.beta) == pytest.approx(ref["best_beta"], abs=1e-12)
        assert rep.best_expectation == pytest.approx(ref["best_expectation"], rel=1e-10)


def test_single_edge_optimum():
    g = Q.Graph.from_edges(2, [(0, 1, 1.0)])
    rep = Q.optimize(g, p=1, budget=300)
    assert abs(rep.best_expectation - 1.0) <= 1e-6


def test_beats_uniform_and_deterministic():
    ratios, uniform = [], []
    for seed in range(4):
        g = Q.random_regular_graph(10, 3, seed=seed)
        rep = Q.optimize(g, p=3, budget=400, seed=seed)
        ratios.append(Q.approximation_ratio(g, rep.best_expectation))
        uniform.append(Q.approximation_ratio(g, Q.expectation(g, Q.init_uniform(10))))
    assert sum(ratios) > sum(uniform)
    g = Q.random_regular_graph(10, 3, seed=0)
    a = Q.optimize(g, p=2, budget=200, seed=0)
    b = Q.optimize(g, p=2, budget=200, seed=0)
    assert a.best_params == b.best_params and a.history == b.history


def test_optimizer_errors():
    g = Q.random_regular_graph(6, 3, seed=0)
    with pytest.raises(ValueError):
        Q.optimize(g, p=1, budget=0)
    with pytest.raises(ValueError):
        Q.optimize(g, p=0)
    with pytest.raises(ValueError):
        Q.optimize(g, p=1, init_strategy="bogus")
    assert Q.approximation_ratio(Q.Graph.from_edges(3, []), 0.0) == 1.0


def test_symmetric_evaluations_match_full_state():
    """N >= 13 optimizer runs evaluate on the psi(x) == psi(~x) half state by
    default; the Nelder-Mead history equals the full-state run's within 1e-10."""
    g = Q.random_regular_graph(16, 3, seed=4)
    a = Q.optimize(g, p=2, budget=60, seed=1, symmetric=True)
    b = Q.optimize(g, p=2, budget=60, seed=1, symmetric=False)
    assert a.evaluations == b.evaluations == 60
    for (i, v), (j, w) in zip(a.history, b.history):
        assert i == j and v == pytest.approx(w, rel=1e-10)
    assert a.best_expectation == pytest.approx(b.best_expectation, rel=1e-10)
