"""The sweep planner (csrc/qaoa_capi.cu make_sets / make_plan) checked on the
CPU through qaoa_plan: for every size class and depth, replaying the plan
symbolically applies cost_l and then RX_l to every qubit exactly once per
level, in circuit order (reference circuit.py:97-113); the fast schedule
merges level boundaries ((R-1)p+1 sweeps); the exact schedule keeps increasing
qubit order; the sharded schedule places one exchange per level right after
the low set."""

import ctypes

import numpy as np
import pytest

from paper_2312_03019_b200 import _lib

EXACT, SHARDED = _lib.RUN_EXACT, _lib.RUN_SHARDED


def plan(n, p, flags):
    L = _lib.load()
    cnt = L.qaoa_plan(n, p, flags, None, 0)
    assert cnt > 0
    out = (ctypes.c_int * (7 * cnt))()
    assert L.qaoa_plan(n, p, flags, out, cnt) == cnt
    return np.array(out, dtype=np.int64).reshape(cnt, 7)


def mixed(carry, q):
    return list(range(12)) if carry >= 12 else list(range(q, q + 12 - carry))


def replay(n, p, rows):
    """Event list: ('cost', l) / ('rx', l, qubit) / ('x', l) in sweep order."""
    ev = []
    for carry, q, pre, s1, mid, s2, ex in rows:
        if pre >= 0:
            ev.append(("cost", pre))
        if s1 >= 0:
            ev += [("rx", s1, b) for b in mixed(carry, q)]
        if mid >= 0:
            ev.append(("cost", mid))
        if s2 >= 0:
            ev += [("rx", s2, b) for b in mixed(carry, q)]
        if ex >= 0:
            ev.append(("x", ex))
    return ev


@pytest.mark.parametrize("n", [12, 13, 16, 20, 21, 22, 26, 30, 33, 36, 40])
@pytest.mark.parametrize("p", [1, 2, 3, 10])
@pytest.mark.parametrize("flags", [0, EXACT, SHARDED, SHARDED | EXACT])
def test_plan_is_the_circuit(n, p, flags):
    rows = plan(n, p, flags)
    ev = replay(n, p, rows)
    costs = [e[1] for e in ev if e[0] == "cost"]
    assert costs == list(range(p))  # one cost per level, in order
    for l in range(p):
        i_cost = ev.index(("cost", l))
        rx = [e for e in ev if e[0] == "rx" and e[1] == l]
        assert sorted(b for _, _, b in rx) == list(range(n))  # every qubit exactly once
        first = min(i for i, e in enumerate(ev) if e[0] == "rx" and e[1] == l)
        last = max(i for i, e in enumerate(ev) if e[0] == "rx" and e[1] == l)
        assert first > i_cost  # cost before the mixer
        if l + 1 < p:
            assert last < ev.index(("cost", l + 1))  # mixer done before the next cost
        if flags & EXACT:
            assert [b for _, _, b in rx] == list(range(n))  # reference qubit order
    # carried bits are never mixed, tiles are 12 bits, runs >= 128 B
    for carry, q, *_ in rows:
        assert 3 <= carry <= 12 and (carry == 12 or q >= carry)
        assert carry == 12 or q + 12 - carry <= n
    R = len({(c, q) for c, q, *_ in rows})
    if flags & SHARDED:
        ex = [e[1] for e in ev if e[0] == "x"]
        assert ex == list(range(p))  # one exchange per level
        for l in range(p):  # right after the low set of that level
            i_x = ev.index(("x", l))
            assert ev[i_x - 1][0] == "rx" and ev[i_x - 1][1] == l and ev[i_x - 1][2] == 11
    elif not flags & EXACT and R >= 3:
        assert len(rows) == (R - 1) * p + 1  # level-boundary merges
    elif flags & EXACT:
        assert len(rows) == R * p


@pytest.mark.parametrize("n", range(22, 41))
def test_merged_high_sets_have_equal_sizes(n):
    """make_sets gives the extra qubits to the middle high sets first, so the
    two sets merged at level boundaries (the first and last high sets) have the
    same size -- the condition of the swapped qubit layout -- except with two
    high sets and an odd remainder (N = 23, 25, 27, 29)."""
    rows = plan(n, 4, 0)
    sets = sorted({(q, carry) for carry, q, *_ in rows if carry < 12})
    sizes = [12 - carry for _, carry in sets]
    assert sum(sizes) == n - 12 and max(sizes) <= 9
    assert max(sizes) - min(sizes) <= 1
    if len(sizes) >= 3 or (n - 12) % 2 == 0:
        assert sizes[0] == sizes[-1]
    # the merged sweeps are exactly the first and last high sets
    merged = {(q, carry) for carry, q, pre, s1, mid, s2, ex in rows if s2 >= 0}
    assert merged == {sets[0], sets[-1]}
