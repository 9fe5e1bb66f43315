"""Small workload touching every kernel variant, for compute-sanitizer
(memcheck / racecheck / synccheck) runs on the GPU box:
    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2312_03019_b200 as Q
from paper_2312_03019_b200.sharded import CudaShard, LocalExchanger, simulate_sharded

for n in (5, 12, 13, 15, 16, 21):
    g = Q.random_regular_graph(n, 3, seed=n) if n % 2 == 0 else Q.erdos_renyi_graph(n, 0.3, n)
    for exact in (True, False):
        pr = Q.QaoaParams((0.3, 1.2, 2.2), (0.5, 2.9, 1.1))
        s = Q.simulate(g, pr, "bitwise", exact=exact, max_qubits=30)
        Q.expectation(g, s)
    Q.build_cut_table(g)
    Q.apply_mixer_layer(s, 0.3)
    Q.apply_cost_layer(s, g, 0.4, "bitwise")
    Q.apply_rx(s, n - 1, 0.2)
# swapped qubit layout: out-of-place low-set sweeps (n = 22: high sets 5 + 5)
g = Q.random_regular_graph(22, 3, seed=2)
s = Q.init_uniform(22, max_qubits=22)
s.engine().call("qaoa_set_layout_swap", 1)
s = Q.simulate(g, Q.QaoaParams((0.3, 1.2), (0.5, 2.9)), "bitwise", max_qubits=22, state=s)
Q.expectation(g, s)
# symmetric half state: mirror low set (fused, merged at two sets and flow 1 at
# three) and the segmented exact run with its mirror passes
for n in (18, 24):
    g = Q.random_regular_graph(n, 3, seed=n)
    pr = Q.QaoaParams((0.3, 1.2, 2.2), (0.5, 2.9, 1.1))
    for exact in (False, True):
        s = Q.simulate(g, pr, "bitwise", exact=exact, symmetric=True, max_qubits=n)
        Q.expectation(g, s)
g = Q.random_regular_graph(16, 3, seed=1)
shards = [CudaShard(14, r) for r in range(4)]
simulate_sharded(g, Q.QaoaParams((0.3, 1.0), (2.9, 0.4)), shards, LocalExchanger(shards), 2)
print("sanitize workload done")
