"""Does RUN_TIMING (an event between sweeps) cost time?  Interleaved A/B of
qaoa_run_layers with and without it at N=30 p=10 (bench workload)."""
import subprocess, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2312_03019_b200 as Q
from paper_2312_03019_b200 import _lib

n, p = 30, 10
g = Q.random_regular_graph(n, 3, seed=0)
tables, cs, ss = Q.level_arrays(g, Q.params_from_seed(p, 0))
stream = torch.cuda.Stream(0)
eng = Q.Engine(n, 0, stream=stream.cuda_stream)
eng.ensure_graph(g)
base = _lib.RUN_EXPECTATION


def run(flags):
    eng.call("qaoa_run_layers", p, _lib.dptr(tables.view(np.float64)), _lib.dptr(cs), _lib.dptr(ss), flags)


for _ in range(3):
    run(base)
ms = int(sys.argv[1]) if len(sys.argv) > 1 else 0
smi = None
if ms:  # bench.py's clock sampler at this polling period
    smi = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw",
                            "--format=csv,noheader,nounits", "-lms", str(ms)],
                           stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
res = {"timing": [], "plain": [], "wall_plain": []}
for rep in range(6):
    for name, fl in (("timing", base | _lib.RUN_TIMING), ("plain", base)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record(stream)
        for _ in range(3):
            run(fl)
        b.record(stream)
        torch.cuda.synchronize()
        res[name].append(a.elapsed_time(b) / 3)
        if name == "plain":
            res["wall_plain"].append((time.perf_counter() - t0) * 1e3 / 3)
for k, v in res.items():
    print(k, [round(x, 2) for x in v], "median", round(float(np.median(v)), 2))
if smi:
    smi.terminate()
