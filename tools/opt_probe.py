"""Optimizer throughput (dev tool): Nelder-Mead evaluations/s with the device-
resident inner loop.   python tools/opt_probe.py N p budget [symmetric 0/1]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_03019_b200 as Q

n, p, budget = (int(x) for x in sys.argv[1:4])
sym = bool(int(sys.argv[4])) if len(sys.argv) > 4 else None
g = Q.random_regular_graph(n, 3, seed=0)
Q.optimize(g, p, budget=5, max_qubits=n, symmetric=sym)  # warm-up (module load, allocation)
t0 = time.perf_counter()
rep = Q.optimize(g, p, budget=budget, max_qubits=n, symmetric=sym)
dt = time.perf_counter() - t0
print(f"N={n} p={p} symmetric={sym}: {rep.evaluations} evaluations in {dt:.2f} s = {rep.evaluations / dt:.0f} evals/s, "
      f"best <C> {rep.best_expectation:.6f}")
