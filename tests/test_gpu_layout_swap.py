"""Swapped qubit layout (qaoa_set_layout_swap, qaoa_capi.cu plan_swaps): every
low-set sweep writes its tiles out of place with the bit ranges of the two
alternately merged high sets exchanged.  Same arithmetic at other addresses, so
the amplitudes must be bit-identical to the in-place run; <C> agrees up to the
order its per-tile partials are summed in."""

import ctypes

import numpy as np
import pytest

import paper_2312_03019_b200 as Q
from paper_2312_03019_b200 import _lib

pytestmark = pytest.mark.gpu


def _run(eng, g, params, mode, flags=0):
    eng.call("qaoa_set_layout_swap", mode)
    tables, cs, ss = Q.level_arrays(g, params)
    t = np.ascontiguousarray(tables)
    eng.call("qaoa_run_layers", params.p, _lib.dptr(t.view(np.float64)), _lib.dptr(cs),
             _lib.dptr(ss), flags | _lib.RUN_EXPECTATION)
    return eng.scalar("qaoa_expectation")


def _state(eng, n):
    import torch

    from paper_2312_03019_b200.state import _wrap_device

    return _wrap_device(eng.state_ptr(), 16 << n, 0).view(torch.complex128).clone()


def _stats(eng):
    nl, hb = ctypes.c_int(), ctypes.c_double()
    _lib.load().qaoa_last_run_stats(eng.ptr, ctypes.byref(nl), ctypes.byref(hb))
    return nl.value, hb.value


@pytest.mark.parametrize("n", [22, 23, 24])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_swapped_layout_bit_identical(n, p):
    """n = 22 / 24: high sets 5+5 / 6+6 (swap applies); n = 23: 6+5 (it does
    not, mode 1 must fall back to in place).  Angle seeds mix both RX forms."""
    import torch

    g = Q.random_regular_graph(n, 3, seed=1) if n % 2 == 0 else \
        Q.erdos_renyi_graph(n, 0.2, seed=1)
    eng = Q.Engine(n)
    try:
        eng.ensure_graph(g)
        for seed in (0, 3):
            params = Q.params_from_seed(p, seed)
            e0 = _run(eng, g, params, 0)
            s0, st0 = _state(eng, n), _stats(eng)
            e1 = _run(eng, g, params, 1)
            s1, st1 = _state(eng, n), _stats(eng)
            assert torch.equal(s0, s1), (n, p, seed)
            assert e1 == pytest.approx(e0, rel=1e-13, abs=1e-13)
            assert st0 == st1
    finally:
        eng.close()


def test_swapped_layout_continuation_and_expect_only():
    """FROM_STATE continuation (a complement mask carried in) and an
    expectation-only last sweep through the swapped layout."""
    import torch

    n = 24
    g = Q.random_regular_graph(n, 3, seed=2)
    eng = Q.Engine(n)
    try:
        eng.ensure_graph(g)
        pa, pb = Q.params_from_seed(3, 5), Q.params_from_seed(4, 6)
        out = {}
        for mode in (0, 1):
            _run(eng, g, pa, mode)
            e = _run(eng, g, pb, mode, _lib.RUN_FROM_STATE)
            out[mode] = (_state(eng, n), e)
            e_only = _run(eng, g, pb, mode, _lib.RUN_FROM_STATE | _lib.RUN_EXPECT_ONLY)
            assert np.isfinite(e_only)
        assert torch.equal(out[0][0], out[1][0])
        assert out[1][1] == pytest.approx(out[0][1], rel=1e-13)
    finally:
        eng.close()


def test_swapped_layout_buffer_and_golden():
    """Mode 1 at BASELINE configs[1] (u3r N=26 seed 0, p=4): one extra state
    buffer, allocated once; amplitudes equal the in-place run; <C> is the
    reference's golden 17.687434636566532.  The default policy leaves N=26
    (7-qubit high sets, C = 5) in place."""
    import torch

    n = 26
    g = Q.random_regular_graph(n, 3, seed=0)
    eng = Q.Engine(n)
    try:
        eng.ensure_graph(g)
        params = Q.params_from_seed(4, 0)
        e_in = _run(eng, g, params, 0)
        s_in = _state(eng, n)
        free0 = torch.cuda.mem_get_info()[0]
        _run(eng, g, params, -1)
        assert torch.cuda.mem_get_info()[0] >= free0 - (64 << 20)  # policy: in place here
        e_sw = _run(eng, g, params, 1)
        free1 = torch.cuda.mem_get_info()[0]
        assert free0 - free1 >= 16 << n  # the second buffer
        assert torch.equal(_state(eng, n), s_in)
        assert e_sw == pytest.approx(17.687434636566532, rel=1e-10)
        assert e_in == pytest.approx(17.687434636566532, rel=1e-10)
        free2 = torch.cuda.mem_get_info()[0]
        _run(eng, g, params, 1)
        assert torch.cuda.mem_get_info()[0] >= free2 - (64 << 20)  # reused, not reallocated
    finally:
        eng.close()


def test_swapped_layout_default_at_n30():
    """The bench configuration (u3r N=30, 9-qubit high sets): the default
    policy swaps (second 16 GiB buffer) and gives the in-place <C>."""
    import torch

    n = 30
    g = Q.random_regular_graph(n, 3, seed=0)
    eng = Q.Engine(n)
    try:
        eng.ensure_graph(g)
        params = Q.params_from_seed(3, 0)
        e_in = _run(eng, g, params, 0)
        free0 = torch.cuda.mem_get_info()[0]
        e_pol = _run(eng, g, params, -1)
        assert free0 - torch.cuda.mem_get_info()[0] >= 16 << n
        assert e_pol == pytest.approx(e_in, rel=1e-13)
    finally:
        eng.close()


def test_layout_swap_rejects_bad_mode():
    eng = Q.Engine(14)
    try:
        with pytest.raises(ValueError):
            eng.call("qaoa_set_layout_swap", 2)
    finally:
        eng.close()


def test_host_driven_runs_stay_in_place():
    """Runs driven through qaoa_run_begin / qaoa_run_sweep_range never use the
    swapped layout (only qaoa_run_layers does): every sweep, the low set's
    included, accepts partial tile ranges, and two halves per sweep give the
    swapped qaoa_run_layers result bit for bit."""
    import torch

    n, p = 24, 2
    g = Q.random_regular_graph(n, 3, seed=4)
    params = Q.params_from_seed(p, 2)
    tables, cs, ss = Q.level_arrays(g, params)
    t = np.ascontiguousarray(tables)
    eng = Q.Engine(n)
    try:
        eng.ensure_graph(g)
        _run(eng, g, params, 1)
        ref = _state(eng, n)
        nseg = ctypes.c_int()
        eng.call("qaoa_run_begin", p, _lib.dptr(t.view(np.float64)), _lib.dptr(cs), _lib.dptr(ss),
                 0, ctypes.byref(nseg))
        L = _lib.load()
        i = 0
        while True:
            seg, carry, q, nt = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
            rc = L.qaoa_run_sweep_info(eng.ptr, i, ctypes.byref(seg), ctypes.byref(carry),
                                       ctypes.byref(q), ctypes.byref(nt))
            if rc == _lib.QAOA_E_RANGE:
                break
            half = nt.value // 2
            eng.call("qaoa_run_sweep_range", i, 0, half)
            eng.call("qaoa_run_sweep_range", i, half, nt.value - half)
            i += 1
        eng.call("qaoa_run_end")
        assert torch.equal(_state(eng, n), ref)
        eng.trim()  # frees the second buffer; the next swapped run re-allocates it
        _run(eng, g, params, 1)
        assert torch.equal(_state(eng, n), ref)
    finally:
        eng.close()


def test_swapped_layout_with_partial_complement_mask():
    """A complement mask that is not swap-invariant (bits in only one of the
    two exchanged ranges, as qaoa_set_cmask / qaoa_apply_rx_range can leave)
    is permuted with the data: swapped == in place, and the mask is unchanged
    after the run (even number of swaps)."""
    import torch

    n = 24  # high sets: bits 12..17 and 18..23
    g = Q.random_regular_graph(n, 3, seed=5)
    eng = Q.Engine(n)
    try:
        eng.ensure_graph(g)
        pa, pb = Q.params_from_seed(2, 7), Q.params_from_seed(3, 8)
        cm = (0b101 << 13) | (1 << 4)  # bits 4, 13, 15
        out = {}
        for mode in (0, 1):
            _run(eng, g, pa, 0)
            eng.call("qaoa_set_cmask", cm)
            e = _run(eng, g, pb, mode, _lib.RUN_FROM_STATE)
            m = ctypes.c_uint64()
            eng.call("qaoa_get_cmask", ctypes.byref(m))
            out[mode] = (_state(eng, n), e, m.value)
        assert torch.equal(out[0][0], out[1][0])
        assert out[1][1] == pytest.approx(out[0][1], rel=1e-13)
        assert out[0][2] == out[1][2]
    finally:
        eng.close()
