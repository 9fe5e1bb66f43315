python -m pytest tests/test_gpu_symmetric.py -q -m gpu -x 2>&1 | tail -5
python tools/sym_probe.py 30 10 5 2>&1 | tail -6
python tools/sym_probe.py 26 4 10 2>&1 | tail -6
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, ".")
import paper_2312_03019_b200 as Q
from paper_2312_03019_b200.symmetric import simulate_symmetric
g = Q.random_regular_graph(24, 3, seed=1)
s = simulate_symmetric(g, Q.params_from_seed(3, 0), fused=True)
print("E", s.expectation(g))
PY
timeout 600 compute-sanitizer --tool memcheck python /tmp/san.py 2>&1 | tail -3
timeout 600 compute-sanitizer --tool racecheck python /tmp/san.py 2>&1 | tail -3
timeout 600 compute-sanitizer --tool synccheck python /tmp/san.py 2>&1 | tail -3
