"""Launch-control helpers (qaoa_capi.cu launch_plan_sweep -> launch_gen_aux,
qaoa_sweep.cu basis_table_kernel / gen_table_kernel): the first sweep of a fast
run reads prebuilt per-tile cut bases and a gen x phase table instead of
building the basis per tile and multiplying every amplitude by gen.  The
product is the same cmul_np the sweep formed, so the state must be bit-identical
with the helpers off (QAOA_GEN_AUX=0, read once per process: one subprocess per
setting).  Reference path: circuit.py:42-48 (init_uniform) + cost.py:162-176."""

import hashlib
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2312_03019_b200 as Q
n, p, kind, seed = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
g = (Q.random_regular_graph(n, 3, seed=seed) if kind == "u3r"
     else Q.erdos_renyi_graph(n, 0.5, seed=seed))
params = Q.params_from_seed(p, seed)
s = Q.simulate(g, params, "bitwise", max_qubits=n)
e = Q.expectation(g, s)
print(hashlib.sha256(np.ascontiguousarray(s.amps).tobytes()).hexdigest(), repr(e))
"""


def _run(env_aux, n, p, kind, seed):
    env = dict(os.environ)
    env["QAOA_GEN_AUX"] = env_aux
    out = subprocess.run([sys.executable, "-c", _CHILD, ROOT, str(n), str(p), kind, str(seed)],
                         env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    sha, e = out.stdout.split()[-2:]
    return sha, float(e)


@pytest.mark.parametrize("n,p,kind,seed", [(18, 3, "u3r", 0), (21, 2, "er", 5), (24, 4, "u3r", 1),
                                           (22, 2, "er", 2), (26, 1, "u3r", 3)])
def test_helpers_bit_identical(n, p, kind, seed):
    on = _run("1", n, p, kind, seed)
    off = _run("0", n, p, kind, seed)
    assert on[0] == off[0], (n, p, kind)
    assert on[1] == off[1]


def test_helpers_counted_in_launches():
    """qaoa_last_run_stats counts the two helper kernels (bench.py gpu_launches)."""
    import ctypes

    import numpy as np

    import paper_2312_03019_b200 as Q
    from paper_2312_03019_b200 import _lib

    n, p = 24, 3
    g = Q.random_regular_graph(n, 3, seed=0)
    eng = Q.Engine(n)
    try:
        eng.ensure_graph(g)
        tables, cs, ss = Q.level_arrays(g, Q.params_from_seed(p, 0))
        t = np.ascontiguousarray(tables)
        eng.call("qaoa_run_layers", p, _lib.dptr(t.view(np.float64)), _lib.dptr(cs), _lib.dptr(ss), 0)
        nl, hb = ctypes.c_int(), ctypes.c_double()
        _lib.load().qaoa_last_run_stats(eng.ptr, ctypes.byref(nl), ctypes.byref(hb))
        sweeps = _lib.load().qaoa_plan(n, p, 0, None, 0)
        assert nl.value == sweeps + 2
    finally:
        eng.close()
