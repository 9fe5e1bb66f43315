"""Run one fused simulate for profiling: python tools/prof_run.py N P [exact]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2312_03019_b200 as Q
from paper_2312_03019_b200 import _lib
n, p = int(sys.argv[1]), int(sys.argv[2])
exact = len(sys.argv) > 3 and sys.argv[3] == "exact"
g = Q.random_regular_graph(n, 3, seed=0)
rng = np.random.default_rng(0)
params = Q.QaoaParams(tuple(rng.uniform(0, 6.28, p)), tuple(rng.uniform(0, 3.14, p)))
tables, cs, ss = Q.level_arrays(g, params)
eng = Q.Engine(n)
eng.ensure_graph(g)
flags = _lib.RUN_EXPECTATION | (_lib.RUN_EXACT if exact else 0)
for _ in range(2):
    eng.call("qaoa_run_layers", p, _lib.dptr(tables.view(np.float64)), _lib.dptr(cs), _lib.dptr(ss), flags)
print("expect", eng.scalar("qaoa_expectation"))
