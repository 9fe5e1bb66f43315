"""Per-evaluation cost at small N (dev tool): the optimizer's inner call
(qaoa_run_layers with RUN_EXPECTATION | RUN_EXPECT_ONLY) timed on the host, the
device time of its launches (RUN_TIMING), and the optimizer's evaluations/s.
    python tools/small_n_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2312_03019_b200 as Q
from paper_2312_03019_b200 import _lib

for n, p in [(16, 4), (20, 1), (20, 4), (22, 4), (24, 4)]:
    g = Q.random_regular_graph(n, 3, seed=0)
    params = Q.params_from_seed(p, 0)
    tables, cs, ss = Q.level_arrays(g, params)
    eng = Q.Engine(n)
    eng.ensure_graph(g)
    L = _lib.load()
    for flags, name in [(_lib.RUN_EXPECTATION, "run+<C>"),
                        (_lib.RUN_EXPECTATION | _lib.RUN_EXPECT_ONLY, "expect-only")]:
        def call(extra=0):
            eng.call("qaoa_run_layers", p, _lib.dptr(tables.view(np.float64)), _lib.dptr(cs),
                     _lib.dptr(ss), flags | extra)
            return eng.scalar("qaoa_expectation")
        for _ in range(20):
            call()
        reps = 500
        t0 = time.perf_counter()
        for _ in range(reps):
            call()
        host_us = (time.perf_counter() - t0) / reps * 1e6
        call(_lib.RUN_TIMING)
        import ctypes
        buf = (ctypes.c_float * 256)()
        k = L.qaoa_layer_timings(eng.ptr, buf, 256)
        dev_us = sum(buf[:k]) * 1e3
        print(f"N={n} p={p} {name}: {host_us:.1f} us per call (host), device sweeps {dev_us:.1f} us "
              f"({k} intervals)")
    eng.close()
    t0 = time.perf_counter()
    rep = Q.optimize(g, p, budget=200, max_qubits=n)
    dt = time.perf_counter() - t0
    print(f"N={n} p={p} optimize: {rep.evaluations / dt:.0f} evaluations/s")
