"""Optimizer throughput (dev tool): Nelder-Mead evaluations/s with the device-
resident inner loop.   python tools/opt_probe.py N p budget"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_03019_b200 as Q

n, p, budget = (int(x) for x in sys.argv[1:4])
g = Q.random_regular_graph(n, 3, seed=0)
Q.optimize(g, p, budget=5, max_qubits=n)  # warm-up (module load, allocation)
t0 = time.perf_counter()
rep = Q.optimize(g, p, budget=budget, max_qubits=n)
dt = time.perf_counter() - t0
print(f"N={n} p={p}: {rep.evaluations} evaluations in {dt:.2f} s = {rep.evaluations / dt:.0f} evals/s, "
      f"best <C> {rep.best_expectation:.6f}")
