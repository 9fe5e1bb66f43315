"""Symmetric half-state mode: N qubits in 2^(N-1) amplitudes.

MaxCut QAOA keeps the state invariant under the global bit flip X^N:
* the launch-control start |+>^N is uniform (circuit.py:42-48);
* C(x) = C(~x), so the cost diagonal (cost.py:162-176) is flip-invariant;
* RX on qubit q commutes with X^N, and the reference's butterfly
  (state.py:114-124) gives psi'(~x) the same products as psi'(x), only added
  in the other order, so psi(x) == psi(~x) holds BIT FOR BIT.

The engine therefore stores only the half with the top qubit N-1 = 0: a
context of N-1 local qubits whose graph has N nodes (the top node is a fixed
0 bit, like the shard bits of a sharded state).  RX on the top qubit pairs
stored y with y ^ (2^(N-1) - 1).  Every run is one `qaoa_run_layers(...,
QAOA_RUN_MIRROR)` call whose tiles fold the virtual qubit in: virtual index v
is stored at v or ~v, so a tile containing qubit N-1 is two sets of stored
runs, the second read backwards.  The fast schedule uses the "mirror low set"
(stored block u of 2048 amplitudes plus block ~u = the virtual tile of qubits
0..10 and N-1; the high sets take 11..N-2); the exact schedule folds qubit N-1
into the top set, after that set's qubits (the reference applies qubit N-1
last).  A level costs the sweeps of a full state of half the size.  The older
segmented form (one `qaoa_mirror_rx` pass per level at the exchange points of
`qaoa_run_begin(..., QAOA_RUN_SHARDED | QAOA_RUN_MIRROR)`) stays available as
``fused=False``.  <C> and the
norm of the full state are twice the half's.  Every amplitude of the full
state is available (`.amps` mirrors the half).

Half the HBM bytes and half the arithmetic per level; N=34 fits one B200.
Opt-in (``simulate(..., symmetric=True)``), launch control; weighted graphs
(the weighted cost is flip-symmetric too) in the fast schedule.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .graph import Graph
from .state import Engine, StateVector, _wrap_device, write_counter


class SymmetricState(StateVector):
    """An N-qubit state stored as its x_{N-1} = 0 half (psi(x) == psi(~x))."""

    __slots__ = ()

    def __init__(self, n: int, engine: Engine):
        StateVector.__init__(self, n, engine=engine)
        engine.call("qaoa_set_mirror", 1)  # sampling walks the 2^n virtual indices

    @property
    def half_engine(self) -> Engine | None:
        return self._eng if self._where == "device" and self._eng is not None \
            and self._eng.n == self.n - 1 else None

    @property
    def amps(self) -> np.ndarray:
        he = self.half_engine
        if he is not None:
            half = he.read()  # true order of the x_top = 0 half
            self._host = np.concatenate([half, half[::-1]])
            self._where = "host"
            self._eng = None  # later engine work takes a full-size context
        return self._host

    @amps.setter
    def amps(self, value: np.ndarray) -> None:
        StateVector.amps.fset(self, value)
        self._eng = None

    def engine(self, device: int = 0) -> Engine:
        """A full-size device copy (the mirrored half appended on the device)."""
        he = self.half_engine
        if he is None:
            return StateVector.engine(self, device)
        import torch

        m = ctypes.c_uint64()
        he.call("qaoa_get_cmask", ctypes.byref(m))
        full = Engine(self.n, he.device)
        h = 1 << (self.n - 1)
        src = _wrap_device(he.state_ptr(), 16 * h, he.device).view(torch.complex128)
        dst = _wrap_device(full.state_ptr(), 16 << self.n, he.device).view(torch.complex128)
        dst[:h].copy_(src)
        dst[h:].copy_(torch.flip(src, [0]))
        torch.cuda.synchronize(he.device)
        full.graph_key = None
        full.call("qaoa_set_cmask", int(m.value))
        he.close()
        self._eng = full
        return full

    def copy(self) -> "StateVector":
        he = self.half_engine
        if he is None:
            return StateVector.copy(self)
        from .state import _copy_device

        m = ctypes.c_uint64()
        he.call("qaoa_get_cmask", ctypes.byref(m))
        eng = Engine(self.n - 1, he.device)
        _copy_device(eng, he.state_ptr(), 16 << (self.n - 1))
        eng.call("qaoa_set_cmask", int(m.value))
        return SymmetricState(self.n, eng)

    def norm(self) -> float:
        he = self.half_engine
        if he is None:
            return StateVector.norm(self)
        return float(np.sqrt(2.0 * he.scalar("qaoa_norm_sq")))

    def expectation(self, g: Graph) -> float:
        he = self.half_engine
        he.ensure_graph(g)
        if not g.is_unweighted:  # float cut values, graph.py:144-151
            he.ensure_weights(g)
            return 2.0 * he.scalar("qaoa_expectation_weighted")
        return 2.0 * he.scalar("qaoa_expectation")


# Runs with at least this many local qubits (every symmetric run) go through
# one qaoa_run_layers call.
FUSED_MIN_LOCAL = 12


def _normalize_top_bit(eng: Engine) -> None:
    """A complement mask with the virtual top bit set describes the same
    stored data as the mask with every bit flipped (psi(x) == psi(~x)): keep
    the top bit clear so reads see the x_top = 0 half."""
    m = ctypes.c_uint64()
    eng.call("qaoa_get_cmask", ctypes.byref(m))
    top = 1 << eng.n
    if m.value & top:
        eng.call("qaoa_set_cmask", int(m.value ^ ((top << 1) - 1)))


def simulate_symmetric(g: Graph, params, exact: bool = False, fuse_expectation: bool = True,
                       state: SymmetricState | None = None, device: int = 0,
                       timing: bool = False, fused: bool | None = None,
                       store_state: bool = True) -> SymmetricState:
    """The p-level circuit on the x_{N-1} = 0 half of the state (see module doc).
    ``fused``: None / True = the one-call schedule; False forces the segmented
    run with one separate mirror pass per level.
    ``store_state=False`` (fused runs with the fused <C>): the last sweep only
    reads; the state may then only give its expectation or be reused as state=."""
    from .circuit import level_arrays

    n = g.n
    if n < 13:
        raise ValueError("the symmetric half-state mode needs at least 13 qubits")
    if not g.is_unweighted and (exact or fused is False):
        raise ValueError("the symmetric half-state mode runs weighted graphs in the fast "
                         "one-call schedule only")
    if fused is None:
        fused = n - 1 >= FUSED_MIN_LOCAL
    he = state.half_engine if isinstance(state, SymmetricState) and state.n == n else None
    eng = he if he is not None else Engine(n - 1, device)
    eng.ensure_graph(g)
    tables, cs, ss = level_arrays(g, params)
    t = np.ascontiguousarray(tables)
    if fused:
        # one call: the low-set sweeps apply the top qubit's RX themselves
        flags = _lib.RUN_MIRROR | (_lib.RUN_EXPECTATION if fuse_expectation else 0) | \
            (_lib.RUN_TIMING if timing else 0) | (_lib.RUN_EXACT if exact else 0)
        if not store_state and fuse_expectation:
            flags |= _lib.RUN_EXPECT_ONLY
        if not g.is_unweighted:
            # factored weighted cost (cost.py:147-159) on the same mirror tiles
            eng.ensure_weights(g)
            gm = np.ascontiguousarray(np.array(params.gamma, dtype=np.float64))
            eng.call("qaoa_run_layers_weighted", params.p, _lib.dptr(gm), _lib.dptr(cs),
                     _lib.dptr(ss), flags)
        else:
            eng.call("qaoa_run_layers", params.p, _lib.dptr(t.view(np.float64)), _lib.dptr(cs),
                     _lib.dptr(ss), flags)
        return _finish(eng, g, params, state, he)
    flags = _lib.RUN_SHARDED | _lib.RUN_MIRROR | (_lib.RUN_EXACT if exact else 0) | \
        (_lib.RUN_EXPECTATION if fuse_expectation else 0) | (_lib.RUN_TIMING if timing else 0)
    nseg = ctypes.c_int()
    eng.call("qaoa_run_begin", params.p, _lib.dptr(t.view(np.float64)), _lib.dptr(cs),
             _lib.dptr(ss), flags, ctypes.byref(nseg))
    L = _lib.load()
    lvl = ctypes.c_int()
    rx = np.zeros(3, dtype=np.float64)
    factor = np.zeros(2, dtype=np.float64)
    for k in range(nseg.value):
        eng.call("qaoa_run_segment", k)
        rc = L.qaoa_run_exchange_info(eng.ptr, k, ctypes.byref(lvl), _lib.dptr(rx), _lib.dptr(factor))
        if rc == _lib.QAOA_E_RANGE:
            continue
        _lib.check(rc)
        eng.call("qaoa_mirror_rx", _lib.dptr(rx), _lib.dptr(factor))
    eng.call("qaoa_run_end")
    return _finish(eng, g, params, state, he)


def _finish(eng: Engine, g: Graph, params, state, he) -> SymmetricState:
    n = g.n
    _normalize_top_bit(eng)
    write_counter.add((1 << n) * (1 + params.p * (n + 1)))
    if state is not None and isinstance(state, SymmetricState) and he is not None:
        return state
    return SymmetricState(n, eng)
