"""Quick GPU parity sweep: engine vs the CPU oracle (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2312_03019_b200 as Q
from oracle import oracle as O

fails = 0
for n in [2, 3, 5, 8, 11, 12, 13, 14, 15, 16, 18, 20, 21, 22]:
    d = 3 if n % 2 == 0 and n > 3 else 2
    g = Q.complete_graph(n) if n < 4 else Q.random_regular_graph(n, d, seed=n)
    for p in (1, 2, 3, 4):
        gm, bt = O.params_from_seed(p, n + p)
        params = Q.QaoaParams(gm, bt)
        ref = O.simulate(n, g.row_mask, g.tot_edge, gm, bt)
        eref = O.expectation(n, g.row_mask, ref)
        for exact in (True, False):
            s = Q.simulate(g, params, "bitwise", exact=exact, max_qubits=30)
            e = Q.expectation(g, s)
            a = s.amps
            diff = np.max(np.abs(a - ref))
            eq = np.array_equal(a, ref)
            rel = abs(e - eref) / max(abs(eref), 1e-300)
            ok = (eq if exact else diff <= 1e-12) and rel <= 1e-10
            if not ok:
                fails += 1
            print(f"n={n:2d} p={p} exact={exact!s:5} eq={eq!s:5} diff={diff:.2e} erel={rel:.1e} {'OK' if ok else 'FAIL'}")
    ct = Q.build_cut_table(g)
    ok = np.array_equal(ct, O.cut_counts(n, g.row_mask))
    fails += not ok
    print(f"n={n} cut table {'OK' if ok else 'FAIL'}")
# single-layer ops
n = 14
g = Q.random_regular_graph(n, 3, seed=1)
rng = np.random.default_rng(0)
amps = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
amps /= np.linalg.norm(amps)
s = Q.StateVector(n, amps.copy())
Q.apply_cost_layer(s, g, 0.7, "bitwise")
Q.apply_mixer_layer(s, 1.1)
r = amps.copy()
O.apply_cost(r, n, g.row_mask, g.tot_edge, 0.7)
O.apply_mixer(r, n, 1.1)
print("single layer eq", np.array_equal(s.amps, r)); fails += not np.array_equal(s.amps, r)
print("FAILS", fails)
