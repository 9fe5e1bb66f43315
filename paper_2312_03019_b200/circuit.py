"""The p-level QAOA circuit on the B200 engine: the drop-in for the reference's
``simulate`` / ``expectation`` (pkg/src/qaoa_maxcut/circuit.py:97-121).

``simulate`` sends the graph's row masks, the host-built phase tables
(cost.py:136-139 expression) and the RX coefficients (state.py:114-115) through
the C ABI ``qaoa_run_layers``: launch-control init, p fused cost+mixer levels
and -- fused into the last sweep -- the expected cut, all in HBM.  The state
comes back device-resident; ``expectation`` returns the fused value when the
state is untouched since, else runs the device reduction.

``exact=True`` reproduces the reference bit for bit (same qubit order and
rounding); the default fast schedule merges adjacent levels' sweeps and uses
one-DFMA butterflies, within 1e-13 of the reference (contract: 1e-12).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cost import phase_table, plan_for
from .graph import Graph
from .state import (
    DEFAULT_MAX_QUBITS,
    Engine,
    StateVector,
    apply_h,
    apply_rx,
    apply_rzz,
    check_qubit_budget,
    init_zero_state,
    write_counter,
)

BACKENDS = ("baseline", "compressed", "bitwise")  # circuit.py:13


@dataclass(frozen=True)
class QaoaParams:
    """Angle schedule: gamma in [0, 2pi), beta in [0, pi), one pair per level."""

    gamma: tuple[float, ...]
    beta: tuple[float, ...]

    def __post_init__(self):
        if len(self.gamma) != len(self.beta):
            raise ValueError("gamma and beta must have the same length")
        if len(self.gamma) < 1:
            raise ValueError("need at least one level")

    @property
    def p(self) -> int:
        return len(self.gamma)


def params_from_seed(p: int, seed: int) -> QaoaParams:
    """Seeded angle schedule of the reference's benchmark harness (bench.py:61-67):
    default_rng(seed), gamma ~ U[0, 2pi) drawn first, then beta ~ U[0, pi)."""
    rng = np.random.default_rng(seed)
    return QaoaParams(
        gamma=tuple(float(v) for v in rng.uniform(0.0, 2.0 * math.pi, p)),
        beta=tuple(float(v) for v in rng.uniform(0.0, math.pi, p)),
    )


def validate_backend(backend: str, g: Graph | None = None) -> str:
    """circuit.py:34-39."""
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}; choose from {BACKENDS}")
    if backend == "bitwise" and g is not None and not g.is_unweighted:
        raise ValueError("bitwise backend requires an unweighted graph")
    return backend


def rx_coefficients(beta: float) -> tuple[float, float]:
    """(cos(theta/2), sin(theta/2)) with theta = -beta (circuit.py:93, state.py:114-115)."""
    theta = -beta
    return math.cos(theta / 2.0), math.sin(theta / 2.0)


def level_arrays(g: Graph, params: QaoaParams):
    """Host-side inputs of qaoa_run_layers: p phase tables and RX coefficients."""
    tables = np.ascontiguousarray(
        np.stack([phase_table(g.tot_edge, gm) for gm in params.gamma]).astype(np.complex128))
    coeffs = [rx_coefficients(b) for b in params.beta]
    cs = np.array([c for c, _ in coeffs], dtype=np.float64)
    ss = np.array([s for _, s in coeffs], dtype=np.float64)
    return tables, cs, ss


def init_uniform(n: int, max_qubits: int = DEFAULT_MAX_QUBITS) -> StateVector:
    """Uniform superposition set directly (launch control, circuit.py:42-48)."""
    check_qubit_budget(n, max_qubits)
    eng = Engine(n)
    eng.call("qaoa_init_uniform")
    write_counter.add(1 << n)
    return StateVector(n, engine=eng)


def init_state(n: int, launch_control: bool = True, threads: int = 1,
               max_qubits: int = DEFAULT_MAX_QUBITS) -> StateVector:
    """circuit.py:51-62: launch control writes the uniform state directly;
    without it, |0..0> and one Hadamard per qubit in increasing order (the
    reference's gate path, same rounding and write count)."""
    if launch_control:
        return init_uniform(n, max_qubits)
    s = init_zero_state(n, max_qubits)
    for q in range(n):
        apply_h(s, q, threads=threads)
    return s


def _init_on(eng: Engine, n: int) -> None:
    """|0..0> plus n Hadamards on an existing engine (launch_control=False)."""
    eng.call("qaoa_init_basis", 0)
    for q in range(n):
        eng.call("qaoa_apply_h", q)
    write_counter.add((n + 1) << n)


def apply_cost_layer(s: StateVector, g: Graph, gamma: float, backend: str = "baseline",
                     threads: int = 1, batch_width: int | None = None,
                     use_table_popcount: bool = False) -> StateVector:
    """One cost layer (circuit.py:65-86): "baseline" = one RZZ(w gamma) pass per
    edge in the graph's edge order (state.py:131-149); the other backends one
    compressed device pass."""
    validate_backend(backend, g)
    from .cost import apply_cost_batched, apply_cost_bitwise, apply_cost_compressed

    if backend == "baseline":
        for i, j, w in g.edges:
            apply_rzz(s, i, j, w * gamma, threads=threads)
        return s
    plan = plan_for(g)
    if not g.is_unweighted:
        return apply_cost_compressed(s, plan, gamma, threads)
    if batch_width is not None and backend == "bitwise":
        return apply_cost_batched(s, plan, gamma, batch_width, use_table_popcount)
    return apply_cost_bitwise(s, plan, gamma, threads)


def apply_mixer_layer(s: StateVector, beta: float, threads: int = 1) -> StateVector:
    """RX(-beta) on every qubit in increasing order (circuit.py:89-94), bit-exact,
    as ceil((n-3)/9) tiled device sweeps."""
    c, sn = rx_coefficients(beta)
    s.engine().call("qaoa_apply_mixer", c, sn)
    write_counter.add(s.n << s.n)
    return s


def simulate(
    g: Graph,
    params: QaoaParams,
    backend: str = "baseline",
    launch_control: bool = True,
    threads: int = 1,
    batch_width: int | None = None,
    use_table_popcount: bool = False,
    max_qubits: int = DEFAULT_MAX_QUBITS,
    *,
    exact: bool = False,
    device: int = 0,
    fuse_expectation: bool = True,
    state: StateVector | None = None,
    store_state: bool = True,
    layout_swap: int | None = None,
    symmetric: bool = False,
) -> StateVector:
    """Run the p-level circuit on the GPU and return the device-resident state
    (circuit.py:97-113).  backend="baseline" (the reference's default) is the
    gate-level path: one device pass per RZZ (edge) and per RX (qubit), bit for
    bit the reference's baseline; "bitwise" / "compressed" run the fused engine.
    launch_control=False starts from |0..0> plus n Hadamards (circuit.py:57-62).

    Extra keyword-only knobs: ``exact`` (bit-exact reference schedule),
    ``device``, ``fuse_expectation`` (accumulate <C> in the last sweep) and
    ``state`` (reuse a StateVector's device buffer instead of allocating) and
    ``symmetric=True`` (unweighted graphs, launch control, N >= 13: store
    only the x_{N-1} = 0 half, psi(x) == psi(~x) bit for bit; see
    ``paper_2312_03019_b200.symmetric``), ``layout_swap`` (-1 / 0 / 1: the swapped-qubit-layout policy of the
    state's engine, see ``Engine.set_layout_swap``; the default policy keeps a
    second 16 B x 2^n device buffer at N=30-type sizes) and
    ``store_state=False`` (only <C> is wanted: the last sweep reads without
    writing back, and the returned state may only be passed to
    ``expectation`` or reused as ``state=``; the optimizer uses it).

    Weighted graphs (backends "compressed" / "baseline", cost.py:147-159): the
    fast schedule runs the same fused sweeps with the weighted cost factored
    per tile (within 1e-12 of the reference); ``exact=True`` (and n < 12) keeps
    the reference's edge-order totals and the exact mixer, bit for bit."""
    validate_backend(backend, g)
    if batch_width is not None and batch_width not in (1, 2, 4, 8):
        raise ValueError(f"batch width must be 1, 2, 4, or 8, got {batch_width}")
    check_qubit_budget(g.n, max_qubits)
    if symmetric:
        if backend == "baseline" or not launch_control:
            raise ValueError("symmetric=True runs the fused engine with launch control")
        from .symmetric import simulate_symmetric

        return simulate_symmetric(g, params, exact=exact, fuse_expectation=fuse_expectation,
                                  state=state, device=device, store_state=store_state)
    if backend == "baseline":
        return _simulate_gates(g, params, launch_control, threads, max_qubits, state)
    if state is not None and state.n == g.n:
        eng = state._eng if state._eng is not None else Engine(g.n, device)
        state._eng, state._host, state._where = eng, None, "device"
        s = state
    else:
        eng = Engine(g.n, device)
        s = StateVector(g.n, engine=eng)
    eng.ensure_graph(g)
    if layout_swap is not None:
        eng.set_layout_swap(layout_swap)
    from_state = 0
    if not launch_control:
        _init_on(eng, g.n)
        from_state = _lib.RUN_FROM_STATE
    if not g.is_unweighted:
        eng.ensure_weights(g)
        if not exact and g.n >= 12 and params.p > 0:
            # fused sweeps with the factored weighted cost (within 1e-12)
            gm = np.ascontiguousarray(np.array(params.gamma, dtype=np.float64))
            cs = np.array([rx_coefficients(b)[0] for b in params.beta], dtype=np.float64)
            ss = np.array([rx_coefficients(b)[1] for b in params.beta], dtype=np.float64)
            wflags = (_lib.RUN_EXPECTATION if fuse_expectation else 0) | from_state
            if not store_state and fuse_expectation:
                wflags |= _lib.RUN_EXPECT_ONLY
            eng.call("qaoa_run_layers_weighted", params.p, _lib.dptr(gm), _lib.dptr(cs),
                     _lib.dptr(ss), wflags)
        else:
            # reference order and rounding: edge-order totals, exact mixer sweeps
            if launch_control:
                eng.call("qaoa_init_uniform")
            for gamma, beta in zip(params.gamma, params.beta):
                eng.call("qaoa_apply_cost_weighted", float(gamma))
                c, sn = rx_coefficients(beta)
                eng.call("qaoa_apply_mixer", c, sn)
        write_counter.add((1 << g.n) * (int(launch_control) + params.p * (g.n + 1)))
        return s
    tables, cs, ss = level_arrays(g, params)
    flags = (_lib.RUN_EXACT if exact else 0) | (_lib.RUN_EXPECTATION if fuse_expectation else 0) \
        | from_state
    if not store_state and fuse_expectation:
        flags |= _lib.RUN_EXPECT_ONLY
    eng.call("qaoa_run_layers", params.p, _lib.dptr(tables.view(np.float64)), _lib.dptr(cs),
             _lib.dptr(ss), flags)
    write_counter.add((1 << g.n) * (int(launch_control) + params.p * (g.n + 1)))
    return s


def _simulate_gates(g: Graph, params: QaoaParams, launch_control: bool, threads: int,
                    max_qubits: int, state: StateVector | None) -> StateVector:
    """The reference's gate-level circuit on the GPU (backend "baseline",
    circuit.py:108-113): init_state, then per level one RZZ pass per edge and
    one RX pass per qubit -- the comparison baseline of run_compare
    (bench.py:184-243), bit-identical to the reference."""
    if state is not None and state.n == g.n and launch_control:
        eng = state._eng if state._eng is not None else Engine(g.n)
        state._eng, state._host, state._where = eng, None, "device"
        eng.call("qaoa_init_uniform")
        write_counter.add(1 << g.n)
        s = state
    else:
        s = init_state(g.n, launch_control, threads, max_qubits)
    for gamma, beta in zip(params.gamma, params.beta):
        apply_cost_layer(s, g, gamma, "baseline", threads)
        for q in range(g.n):
            apply_rx(s, q, -beta, threads=threads)
    return s


def expectation(g: Graph, s: StateVector) -> float:
    """sum_x |amp_x|^2 C(x) on the device (circuit.py:116-121): deterministic
    fixed-order reduction; the fused value of the last simulate when valid."""
    if s.n != g.n:
        raise ValueError(f"state has {s.n} qubits but graph has {g.n} nodes")
    if getattr(s, "half_engine", None) is not None:
        return s.expectation(g)  # symmetric half state: twice the half's sum
    eng = s.engine()
    eng.ensure_graph(g)
    if not g.is_unweighted:  # float cut values, graph.py:144-151
        eng.ensure_weights(g)
        return eng.scalar("qaoa_expectation_weighted")
    return eng.scalar("qaoa_expectation")


def sample(s: StateVector, shots: int, seed: int = 0) -> np.ndarray:
    """Draw basis indices with probability |amp|^2 (circuit.py:124-133) without
    moving the state off the device: the same uniforms as numpy's
    ``default_rng(seed).choice(size, shots, p=probs/total)`` (cdf search,
    side='right'), the cdf evaluated on the GPU per 4096-amplitude block."""
    if shots < 1:
        raise ValueError("shots must be at least 1")
    import ctypes

    # a symmetric half state samples in place (its engine walks the virtual
    # full index space, qaoa_set_mirror) instead of materialising the full state
    eng = getattr(s, "half_engine", None) or s.engine()
    bb = min(s.n - (1 if eng.n < s.n else 0), 12)
    norms = np.empty(1 << (s.n - bb), dtype=np.float64)
    eng.call("qaoa_block_norms", bb, _lib.dptr(norms))
    prefix = np.cumsum(norms)
    total = float(prefix[-1])
    if abs(total - 1.0) > 1e-6:
        raise ValueError(f"state is not normalized (norm^2 = {total!r})")
    u = np.random.default_rng(seed).random(shots)
    targets = u * total
    blk = np.minimum(np.searchsorted(prefix, targets, side="right"), prefix.size - 1)
    order = np.argsort(blk, kind="stable")
    sb = blk[order]
    groups, starts = np.unique(sb, return_index=True)
    offs = np.append(starts, shots).astype(np.int64)
    base = np.where(groups > 0, prefix[np.maximum(groups - 1, 0)], 0.0).astype(np.float64)
    t_sorted = np.ascontiguousarray(targets[order])
    out_sorted = np.empty(shots, dtype=np.int64)
    gblk = np.ascontiguousarray(groups.astype(np.int64))
    eng.call("qaoa_sample_blocks", bb, ctypes.c_int64(groups.size),
             gblk.ctypes.data_as(_lib._i64p), _lib.dptr(base), offs.ctypes.data_as(_lib._i64p),
             _lib.dptr(t_sorted), out_sorted.ctypes.data_as(_lib._i64p))
    out = np.empty(shots, dtype=np.int64)
    out[order] = out_sorted
    return out


def gate_counts(n: int, g: Graph, p: int) -> tuple[int, int, int]:
    """(H, RZZ, RX) counts without launch control (circuit.py:136-138)."""
    return n, p * g.tot_edge, p * n
