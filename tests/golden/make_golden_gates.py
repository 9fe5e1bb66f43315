"""Golden fixtures for the gate-level path, made by running the REFERENCE itself.

Covers the reference's default ``backend="baseline"`` (per-edge RZZ sweeps,
circuit.py:76-80, state.py:131-149), ``launch_control=False`` (|0..0> plus one
Hadamard per qubit, circuit.py:57-62, state.py:66-107) and the single gates
apply_h / apply_rzz on random states.  Run in the build container:
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_gates.py
Outputs (committed): golden_gates.npz, golden_gates.json.  Test time never
reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from qaoa_maxcut import Graph, expectation, random_regular_graph, simulate  # noqa: E402
from qaoa_maxcut.bench import params_from_seed  # noqa: E402
from qaoa_maxcut.circuit import init_state  # noqa: E402
from qaoa_maxcut.graph import complete_graph, cycle_graph  # noqa: E402
from qaoa_maxcut.state import StateVector, apply_h, apply_rzz, write_counter  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"cases": [], "init": [], "gates": []}

    cases = []
    for n in (2, 3, 5, 8, 11, 12, 13):
        g = complete_graph(n) if n < 4 else random_regular_graph(n, 3 if n % 2 == 0 else 2, seed=n)
        cases.append((f"base_rr{n}", g, params_from_seed(2, n), True))
    cases.append(("base_rr10_nolc", random_regular_graph(10, 3, seed=4), params_from_seed(3, 4), False))
    cases.append(("base_cycle9_nolc", cycle_graph(9), params_from_seed(2, 9), False))
    cases.append(("base_w3r12", random_regular_graph(12, 3, weighted=True, seed=2),
                  params_from_seed(2, 2), True))
    cases.append(("base_w3r8_nolc", random_regular_graph(8, 3, weighted=True, seed=5),
                  params_from_seed(3, 5), False))
    for name, g, pr, lc in cases:
        write_counter.reset()
        s = simulate(g, pr, backend="baseline", launch_control=lc, max_qubits=16)
        arrays["amps_" + name] = s.amps.copy()
        meta["cases"].append({
            "name": name, "n": g.n, "edges": [list(e) for e in g.edges],
            "gamma": list(pr.gamma), "beta": list(pr.beta), "launch_control": lc,
            "expectation": float(expectation(g, s)), "amp_writes": int(write_counter.amp_writes),
        })

    for n in (1, 4, 9, 14):
        write_counter.reset()
        s = init_state(n, launch_control=False, max_qubits=16)
        arrays[f"init_nolc_{n}"] = s.amps.copy()
        meta["init"].append({"n": n, "amp_writes": int(write_counter.amp_writes)})

    rng = np.random.default_rng(11)
    n = 10
    a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    arrays["gate_in"] = a.copy()
    s = StateVector(n, a.copy())
    ops = [("h", 0), ("h", 9), ("h", 4), ("rzz", 0, 9, 0.83), ("rzz", 7, 2, -2.1), ("rzz", 3, 4, 5.5),
           ("h", 3)]
    for k, op in enumerate(ops):
        if op[0] == "h":
            apply_h(s, op[1])
        else:
            apply_rzz(s, op[1], op[2], op[3])
        arrays[f"gate_out_{k}"] = s.amps.copy()
        meta["gates"].append(list(op))
    meta["gate_n"] = n

    np.savez_compressed(os.path.join(HERE, "golden_gates.npz"), **arrays)
    with open(os.path.join(HERE, "golden_gates.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
