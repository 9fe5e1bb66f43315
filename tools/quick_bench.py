"""Quick perf probe: per-sweep device times via QAOA_RUN_TIMING (dev tool)."""
import sys, os, time, json, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2312_03019_b200 as Q
from paper_2312_03019_b200 import _lib
from oracle import oracle as O

peak = 6549.1
for n, p in [(int(a.split(':')[0]), int(a.split(':')[1])) for a in (sys.argv[1:] or ["26:4", "30:10"])]:
    g = Q.random_regular_graph(n, 3, seed=0)
    gm, bt = O.params_from_seed(p, 0)
    params = Q.QaoaParams(gm, bt)
    tables, cs, ss = Q.level_arrays(g, params)
    eng = Q.Engine(n)
    eng.ensure_graph(g)
    for exact in (False, True):
        flags = _lib.RUN_EXPECTATION | _lib.RUN_TIMING | (_lib.RUN_EXACT if exact else 0)
        for it in range(int(os.environ.get("QB_ITERS", "3"))):
            t0 = time.perf_counter()
            eng.call("qaoa_run_layers", p, _lib.dptr(tables.view(np.float64)), _lib.dptr(cs), _lib.dptr(ss), flags)
            wall = time.perf_counter() - t0
        ms = (ctypes.c_float * 256)()
        k = _lib.load().qaoa_layer_timings(eng.ptr, ms, 256)
        times = list(ms[:k])
        e = eng.scalar("qaoa_expectation")
        tot = sum(times)
        bw = [32 * 2**n / (t * 1e-3) / 1e9 for t in times]
        print(json.dumps({"n": n, "p": p, "exact": exact, "sweeps": k, "total_ms": round(tot, 3), "wall_ms": round(wall*1e3, 2),
                          "layers_per_s": round(p / (tot * 1e-3), 2), "expect": e,
                          "sweep_ms": [round(t, 3) for t in times[:8]],
                          "sweep_GBps": [round(b) for b in bw[:8]], "frac_first": round(bw[min(1, k-1)] / peak, 3)}))
    eng.close()
