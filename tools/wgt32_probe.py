"""Weighted (compressed backend) fast simulate at N=30, p=4 and p=10 (dev tool):
time per call with the state reused, and <C>.   python tools/wgt32_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2312_03019_b200 as Q

n = 30
g = Q.random_regular_graph(n, 3, seed=0)
rng = np.random.default_rng(1)
wg = Q.Graph.from_edges(n, [(i, j, float(w)) for (i, j, _), w in zip(g.edges, rng.uniform(0.5, 2.0, len(g.edges)))])
for p in (4, 10):
    pr = Q.params_from_seed(p, 0)
    s = Q.simulate(wg, pr, "compressed", max_qubits=n)
    Q.simulate(wg, pr, "compressed", max_qubits=n, state=s)
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        s = Q.simulate(wg, pr, "compressed", max_qubits=n, state=s)
        e = Q.expectation(wg, s)
    dt = (time.perf_counter() - t0) / reps
    print(f"weighted N={n} p={p}: {dt * 1e3:.1f} ms per simulate + <C> = {p / dt:.1f} layers/s, <C> = {e!r}")
