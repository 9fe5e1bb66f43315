"""Symmetric half-state mode timing (tooling): fused (mirror inside the low-set
sweeps) vs segmented (one mirror pass per level), N qubits, p levels, per-launch
CUDA-event times of the fused run."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2312_03019_b200 as Q
from paper_2312_03019_b200 import _lib
from paper_2312_03019_b200.symmetric import simulate_symmetric

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
p = int(sys.argv[2]) if len(sys.argv) > 2 else 10
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
g = Q.random_regular_graph(n, 3, seed=0) if n % 2 == 0 else \
    Q.Graph.from_edges(n, list(Q.random_regular_graph(n - 1, 3, seed=0).edges))
pr = Q.params_from_seed(p, 0)
for fused in (True, False):
    s = simulate_symmetric(g, pr, fused=fused, timing=True)
    for _ in range(2):
        simulate_symmetric(g, pr, state=s, fused=fused, timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        simulate_symmetric(g, pr, state=s, fused=fused, timing=fused)
        e = s.expectation(g)
    dt = (time.perf_counter() - t0) / reps
    line = f"N={n} p={p} fused={fused}: {1e3 * dt:.2f} ms/step = {p / dt:.1f} layers/s, <C>={e!r}"
    if fused:
        buf = (ctypes.c_float * 4096)()
        k = _lib.load().qaoa_layer_timings(s.half_engine.ptr, buf, 4096)
        line += "\n  launches (ms): " + " ".join(f"{x:.3f}" for x in buf[:k])
    print(line, flush=True)
    s.half_engine.close()
