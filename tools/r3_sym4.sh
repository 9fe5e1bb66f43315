python -m pytest tests/test_gpu_symmetric.py tests/test_gpu_optimize.py tests/test_gpu_sanitizers.py -q -m gpu 2>&1 | tail -6
python tools/sym_probe.py 30 10 5 2>&1 | tail -4
python - <<'PY'
import sys, time; sys.path.insert(0, ".")
import torch, paper_2312_03019_b200 as Q
from paper_2312_03019_b200.symmetric import simulate_symmetric
g = Q.random_regular_graph(30, 3, seed=0); pr = Q.params_from_seed(10, 0)
for fused in (True, False):
    s = simulate_symmetric(g, pr, exact=True, fused=fused)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(3): simulate_symmetric(g, pr, exact=True, fused=fused, state=s)
    dt = (time.perf_counter() - t0) / 3
    print(f"exact symmetric N=30 p=10 fused={fused}: {10 / dt:.1f} layers/s, <C>={s.expectation(g)!r}")
    s.half_engine.close()
PY
