"""Kernels for an extra ncu capture (dev tool): one exchange (G=8 virtual
shards, N=28) and one weighted fused simulate (N=28, p=2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2312_03019_b200 as Q
from paper_2312_03019_b200 import sharded as S

n = 28
g = Q.random_regular_graph(n, 3, seed=0)
pr = Q.params_from_seed(2, 0)
shards = [S.CudaShard(n - 3, r) for r in range(8)]
S.simulate_sharded_fused(g, pr, shards, S.PeerExchanger(shards), 3, expect=True)
for s in shards:
    s.close()
rng = np.random.default_rng(1)
wg = Q.Graph.from_edges(n, [(i, j, float(rng.uniform(0.1, 2.0))) for i, j, _ in g.edges])
s = Q.simulate(wg, pr, "compressed", max_qubits=n)
print("weighted <C>", Q.expectation(wg, s))
