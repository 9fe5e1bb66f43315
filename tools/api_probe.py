"""Timing of the secondary public entry points at one size (dev tool):
standalone <C>, single cost layer, single mixer layer (exact sweeps), weighted
(compressed backend) simulate, sampling.   python tools/api_probe.py N"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2312_03019_b200 as Q

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
g = Q.random_regular_graph(n, 3, seed=0)
pr = Q.params_from_seed(2, 0)
s = Q.simulate(g, pr, "bitwise", max_qubits=n)
size_gb = 16 * (1 << n) / 1e9


def t(fn, reps=5):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


ms_rx = t(lambda: Q.apply_rx(s, 0, 0.0))
ms = t(lambda: Q.expectation(g, Q.apply_rx(s, 0, 0.0)))  # RX invalidates the fused <C>
print(f"N={n}: apply_rx(q=0): {ms_rx:.2f} ms = {2 * size_gb / ms_rx:.2f} TB/s; "
      f"standalone <C>: {ms - ms_rx:.2f} ms = {size_gb / (ms - ms_rx):.2f} TB/s")
ms = t(lambda: Q.apply_cost_layer(s, g, 0.7, "bitwise"))
print(f"apply_cost_layer (bitwise): {ms:.2f} ms = {2 * size_gb / ms:.2f} TB/s")
ms = t(lambda: Q.apply_mixer_layer(s, 0.3))
print(f"apply_mixer_layer (exact sweeps): {ms:.2f} ms")
wg = Q.Graph.from_edges(n, [(i, j, 0.5 + ((i * 7 + j) % 5) / 4) for i, j, _ in g.edges])
ws = Q.simulate(wg, pr, "compressed", max_qubits=n)
ms = t(lambda: Q.simulate(wg, pr, "compressed", max_qubits=n, state=ws), reps=3)
ms_u = t(lambda: Q.simulate(g, pr, "bitwise", max_qubits=n, state=ws), reps=3)
ms_x = t(lambda: Q.simulate(wg, pr, "compressed", max_qubits=n, state=ws, exact=True), reps=2)
print(f"simulate p=2, state reused: weighted fused {ms:.2f} ms | unweighted {ms_u:.2f} ms | "
      f"weighted reference-order (exact) {ms_x:.1f} ms")
ms = t(lambda: Q.sample(s, 1000, seed=1), reps=3)
print(f"sample 1000 shots: {ms:.2f} ms")
