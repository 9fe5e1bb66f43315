"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
Outputs (committed): golden_small.npz, golden_meta.json.  Nothing at test time
reads /root/reference; the tests read these files.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from qaoa_maxcut import (  # noqa: E402  (reference package)
    Graph,
    QaoaParams,
    expectation,
    random_regular_graph,
    simulate,
)
from qaoa_maxcut.graph import complete_graph, cycle_graph  # noqa: E402
from qaoa_maxcut.bench import params_from_seed  # noqa: E402
from qaoa_maxcut.cost import (  # noqa: E402
    _phase_table,
    apply_cost_bitwise,
    plan_for,
    row_cut_count,
)
from qaoa_maxcut.circuit import apply_mixer_layer  # noqa: E402
from qaoa_maxcut.state import StateVector  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def acceptance_graph(rng: np.random.Generator) -> Graph:
    """test_acceptance.py:46-57 (_random_graph), unweighted draws."""
    n = int(rng.integers(2, 13))
    edges = []
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < 0.4:
                edges.append((i, j, 1.0))
    if not edges:
        edges.append((0, 1, 1.0))
    return Graph.from_edges(n, edges)


def er_graph(n: int, p: float, seed: int) -> Graph:
    """SURVEY.md section 8d ER pattern (the reference's test_acceptance.py loop)."""
    rng = np.random.default_rng(seed)
    return Graph.from_edges(n, [(i, j, 1.0) for i in range(n) for j in range(i + 1, n)
                                if rng.random() < p])


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"cases": [], "big": [], "graphs": {}, "params": {}, "kat": {}}

    # --- full-amplitude cases (small n): simulate(bitwise) ---------------------
    cases = []
    for n in range(2, 13):
        g = complete_graph(n) if n < 4 else random_regular_graph(n, 3 if n % 2 == 0 else 2, seed=n)
        cases.append((f"rr{n}", g, params_from_seed(3, n)))
    cases.append(("triangle_p2", Graph.from_edges(3, [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0)]),
                   params_from_seed(2, 7)))
    cases.append(("complete10_p2", complete_graph(10), params_from_seed(2, 3)))
    cases.append(("cycle9_p4", cycle_graph(9), params_from_seed(4, 9)))
    rng = np.random.default_rng(1)
    for k in range(12):
        g = acceptance_graph(rng)
        p = int(rng.integers(1, 6))
        pr = QaoaParams(gamma=tuple(rng.uniform(0.0, 2 * math.pi, p)),
                        beta=tuple(rng.uniform(0.0, math.pi, p)))
        cases.append((f"accept{k}", g, pr))
    for name, g, pr in cases:
        s = simulate(g, pr, "bitwise")
        arrays[f"amps_{name}"] = s.amps
        arrays[f"cut_{name}"] = plan_for(g).cut_counts()
        meta["cases"].append({
            "name": name, "n": g.n, "edges": [[i, j] for i, j, _ in g.edges],
            "tot_edge": g.tot_edge, "gamma": list(pr.gamma), "beta": list(pr.beta),
            "expectation": expectation(g, s),
        })

    # --- weighted graphs: the "compressed" backend (cost.py:147-159) -----------
    meta["weighted"] = []
    wcases = [(f"w3r{n}", random_regular_graph(n, 3, weighted=True, seed=n), params_from_seed(3, n))
              for n in (6, 8, 10, 12, 14)]
    rngw = np.random.default_rng(2)
    for k in range(8):
        n = int(rngw.integers(2, 13))
        edges = [(i, j, float(rngw.uniform(0.1, 1.0))) for i in range(n) for j in range(i + 1, n)
                 if rngw.random() < 0.4] or [(0, 1, 0.5)]
        p = int(rngw.integers(1, 5))
        pr = QaoaParams(gamma=tuple(rngw.uniform(0.0, 2 * math.pi, p)),
                        beta=tuple(rngw.uniform(0.0, math.pi, p)))
        wcases.append((f"wacc{k}", Graph.from_edges(n, edges), pr))
    for name, g, pr in wcases:
        s = simulate(g, pr, "compressed")
        arrays[f"wamps_{name}"] = s.amps
        meta["weighted"].append({
            "name": name, "n": g.n, "edges": [[i, j, w] for i, j, w in g.edges],
            "gamma": list(pr.gamma), "beta": list(pr.beta), "expectation": expectation(g, s),
        })

    # --- single cost layer / mixer layer on a random state (n = 10) ------------
    g = random_regular_graph(10, 3, seed=4)
    r = np.random.default_rng(5)
    amps = r.normal(size=1 << 10) + 1j * r.normal(size=1 << 10)
    amps /= np.linalg.norm(amps)
    arrays["layer_in"] = amps.copy()
    s = StateVector(10, amps.copy())
    apply_cost_bitwise(s, plan_for(g), 0.7)
    arrays["layer_cost_out"] = s.amps.copy()
    apply_mixer_layer(s, 1.1)
    arrays["layer_mix_out"] = s.amps.copy()
    meta["layer"] = {"n": 10, "edges": [[i, j] for i, j, _ in g.edges], "gamma": 0.7, "beta": 1.1}

    # --- larger n: hashes + <C> + a strided sample -----------------------------
    for n, p in ((16, 2), (18, 4), (20, 1), (20, 3), (22, 4)):
        g = random_regular_graph(n, 3, seed=0)
        pr = params_from_seed(p, 0)
        s = simulate(g, pr, "bitwise", max_qubits=30)
        idx = np.arange(0, 1 << n, 997)
        key = f"u3r{n}_p{p}"
        arrays[f"sample_{key}"] = s.amps[idx]
        meta["big"].append({
            "key": key, "n": n, "p": p, "seed": 0, "expectation": expectation(g, s),
            "amps_sha256": sha(s.amps), "cut_sha256": sha(plan_for(g).cut_counts()),
            "sample_stride": 997, "norm2": float(np.sum(np.abs(s.amps) ** 2)),
        })
    ger = er_graph(14, 0.5, 0)
    meta["graphs"]["er14_seed0"] = [[i, j] for i, j, _ in ger.edges]
    arrays["cut_er14"] = plan_for(ger).cut_counts()

    # --- generators and angle schedules ----------------------------------------
    for n, seed in ((20, 0), (26, 0), (30, 0), (32, 0), (36, 0), (10, 3), (8, 1)):
        meta["graphs"][f"u3r{n}_seed{seed}"] = [[i, j] for i, j, _ in random_regular_graph(n, 3, seed=seed).edges]
    meta["graphs"]["er33_seed0"] = [[i, j] for i, j, _ in er_graph(33, 0.5, 0).edges]
    for p in (1, 4, 10):
        pr = params_from_seed(p, 0)
        meta["params"][f"p{p}_seed0"] = {"gamma": list(pr.gamma), "beta": list(pr.beta)}

    # --- known-answer tests the reference's own tests assert -------------------
    meta["kat"]["row_step"] = list(row_cut_count(0b00010110, 0b00001011, 1, word_bits=8))
    meta["kat"]["phase_table_E3_g0.9"] = [[float(v.real), float(v.imag)] for v in _phase_table(3, 0.9)]
    arrays["phase_table_E45"] = _phase_table(45, 4.002148315014479)
    # <C> reference values quoted in SURVEY.md Appendix B (N=26 p=4 run here too)
    g26 = random_regular_graph(26, 3, seed=0)
    plan_for(g26).cut_counts()
    s26 = simulate(g26, params_from_seed(4, 0), "bitwise", max_qubits=26, threads=8)
    meta["big"].append({"key": "u3r26_p4", "n": 26, "p": 4, "seed": 0,
                        "expectation": expectation(g26, s26), "amps_sha256": sha(s26.amps),
                        "sample_stride": 99991, "norm2": float(np.sum(np.abs(s26.amps) ** 2))})
    arrays["sample_u3r26_p4"] = s26.amps[np.arange(0, 1 << 26, 99991)]

    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **arrays)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", len(arrays), "arrays;", len(meta["cases"]), "cases;", len(meta["big"]), "big")


if __name__ == "__main__":
    main()
