"""Run the symmetric half-state schedule for profiling (tooling):
python tools/prof_sym.py N P -- two fused runs (mirror low set + high sets)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_03019_b200 as Q
from paper_2312_03019_b200.symmetric import simulate_symmetric

n, p = int(sys.argv[1]), int(sys.argv[2])
g = Q.random_regular_graph(n, 3, seed=0)
pr = Q.params_from_seed(p, 0)
s = simulate_symmetric(g, pr)
s = simulate_symmetric(g, pr, state=s)
print("expect", s.expectation(g))
