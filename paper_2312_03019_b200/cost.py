"""Cost-layer surface: the bitwise cut table and the compressed (one-pass) cost layer.

Mirrors the reference's cost module (pkg/src/qaoa_maxcut/cost.py):
``CompressedCostPlan`` / ``plan_for`` (cost.py:66-108) with ``cut_counts``
built on the GPU by the bitwise kernel (K1, bit-exact), the phase table
``_phase_table`` built on the host with the reference's numpy expression
(cost.py:136-139, so the table is bit-identical), and ``apply_cost_bitwise``
(cost.py:162-176) as one device pass.  The scalar bitwise primitives
(cost.py:26-63, :111-133) are host helpers with the same results.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

from . import _lib
from .graph import MASK_BITS, Graph
from .state import Engine, StateVector, write_counter


def phase_table(tot_edge: int, gamma: float) -> np.ndarray:
    """exp(-i gamma t / 2) for t = -E..E; entry t+E (cost.py:136-139, same expression)."""
    levels = np.arange(-tot_edge, tot_edge + 1, dtype=np.float64)
    return np.exp(-0.5j * gamma * levels)


_phase_table = phase_table


def popcount_int(value: int, use_table: bool = False) -> int:
    """Set bits of a Python int (cost.py:39-46; the LUT variant gives the same count)."""
    return int(value).bit_count()


def popcount_u64(values: np.ndarray, use_table: bool = False) -> np.ndarray:
    """Set bits per uint64 element (cost.py:26-36)."""
    return np.bitwise_count(np.ascontiguousarray(values, dtype=np.uint64))


def broadcast_bit(b: int, i: int, word_bits: int = MASK_BITS) -> int:
    """All-ones word iff bit i of b is set (two's complement, cost.py:49-52)."""
    return ((1 << word_bits) - 1) if (b >> i) & 1 else 0


def row_cut_count(b: int, row_mask: int, i: int, word_bits: int = MASK_BITS,
                  use_table: bool = False) -> tuple[int, int, int, int]:
    """(b_I, b_I ^ b, row_mask & (b_I ^ b), popcount): one row of Alg. 3 (cost.py:55-63)."""
    bi = broadcast_bit(b, i, word_bits)
    xored = (bi ^ b) & ((1 << word_bits) - 1)
    masked = row_mask & xored
    return bi, xored, masked, masked.bit_count()


class CompressedCostPlan:
    """Per-graph cost plan (cost.py:66-108).  ``cut_counts`` is produced by the
    GPU cut-table builder (K1) and cached on the host, like the reference's
    lazily built int64 table."""

    def __init__(self, graph: Graph):
        self.graph = graph
        self.row_mask = np.array(graph.row_mask, dtype=np.uint64)
        self.tot_edge = graph.tot_edge
        self.weights = tuple(w for _, _, w in graph.edges)
        self._cut_counts: np.ndarray | None = None
        self._rotation_totals: np.ndarray | None = None

    def rotation_totals(self) -> np.ndarray:
        """Signed rotation total sum_e w_e (1 - 2 [x_i != x_j]) per basis index,
        float64, accumulated in edge order on the GPU (cost.py:77-86; bit-identical)."""
        if self._rotation_totals is None:
            self._rotation_totals = edge_values(self.graph, 0)
        return self._rotation_totals

    def _require_unweighted(self) -> None:
        if not self.graph.is_unweighted:
            raise ValueError("bitwise cost kernel requires an unweighted graph")

    def cut_counts(self) -> np.ndarray:
        """int64 C(x) for every x in [0, 2^n) (cost.py:88-99), built on the GPU."""
        if self._cut_counts is None:
            self._require_unweighted()
            self._cut_counts = build_cut_table(self.graph)
        return self._cut_counts


@lru_cache(maxsize=128)
def plan_for(graph: Graph) -> CompressedCostPlan:
    return CompressedCostPlan(graph)


def build_cut_table(g: Graph, device: int = 0) -> np.ndarray:
    """Run the GPU bitwise cut-table kernel and return the table as int64."""
    eng = Engine(g.n, device)
    try:
        eng.ensure_graph(g)
        eng.call("qaoa_build_cut_table")
        out = np.empty(1 << g.n, dtype=np.int64)
        eng.call("qaoa_read_cut_table", 0, out.size, out.ctypes.data_as(_lib._i64p))
        return out
    finally:
        eng.close()


def edge_values(g: Graph, kind: int, device: int = 0) -> np.ndarray:
    """Per-index float64 edge sums in edge order, computed on the GPU
    (qaoa_edge_values): kind 0 = rotation totals (cost.py:77-86), kind 1 = cut
    values (graph.py:144-151)."""
    eng = Engine(g.n, device)
    try:
        eng.ensure_weights(g)
        out = np.empty(1 << g.n, dtype=np.float64)
        eng.call("qaoa_edge_values", int(kind), 0, out.size, _lib.dptr(out))
        return out
    finally:
        eng.close()


def cut_edge_count_bitwise(plan: CompressedCostPlan, b: int, use_table: bool = False) -> int:
    """Cut edges of assignment b from per-row popcounts (cost.py:122-128)."""
    plan._require_unweighted()
    return sum(row_cut_count(b, plan.graph.row_mask[i], i)[3] for i in range(plan.graph.n))


def total_rotation_unweighted(plan: CompressedCostPlan, b: int) -> int:
    """E - 2 C(b) (cost.py:131-133)."""
    return plan.tot_edge - 2 * cut_edge_count_bitwise(plan, b)


def total_rotation_weighted(plan: CompressedCostPlan, b: int) -> float:
    """sum_e w_e (-1)^(b_i xor b_j) (cost.py:111-119)."""
    total = 0.0
    for i, j, w in plan.graph.edges:
        total += -w if ((b >> i) ^ (b >> j)) & 1 else w
    return total


def _check_state(s: StateVector, plan: CompressedCostPlan) -> None:
    if s.n != plan.graph.n:
        raise ValueError(f"state has {s.n} qubits but graph has {plan.graph.n} nodes")


def apply_cost_bitwise(s: StateVector, plan: CompressedCostPlan, gamma: float,
                       threads: int = 1) -> StateVector:
    """amp[x] *= table[E - 2 C(x) + E] in one device pass, C(x) recomputed on the
    fly from the row masks (cost.py:162-176).  Bit-exact with the reference."""
    _check_state(s, plan)
    plan._require_unweighted()
    table = np.ascontiguousarray(phase_table(plan.tot_edge, gamma))
    eng = s.engine()
    eng.ensure_graph(plan.graph)
    eng.call("qaoa_apply_cost", _lib.dptr(table.view(np.float64)))
    write_counter.add(1 << s.n)
    return s


def apply_cost_compressed(s: StateVector, plan: CompressedCostPlan, gamma: float,
                          threads: int = 1) -> StateVector:
    """Weighted rotation-compressed cost layer, one device pass (cost.py:147-159):
    amp *= exp(-i gamma t(x) / 2) with t accumulated in edge order.  Unweighted
    graphs take the bit-exact integer path (same values, test_cost.py:153-162)."""
    _check_state(s, plan)
    if plan.graph.is_unweighted:
        return apply_cost_bitwise(s, plan, gamma, threads)
    eng = s.engine()
    eng.ensure_graph(plan.graph)
    eng.ensure_weights(plan.graph)
    eng.call("qaoa_apply_cost_weighted", float(gamma))
    write_counter.add(1 << s.n)
    return s


def apply_cost_batched(s: StateVector, plan: CompressedCostPlan, gamma: float, batch_width: int,
                       use_table_popcount: bool = False) -> StateVector:
    """Strip-mined variant (cost.py:179-218): the warp is the strip on the GPU, so
    this is the same device pass as ``apply_cost_bitwise`` (results identical,
    as the reference requires, test_cost.py:186-195)."""
    if batch_width not in (1, 2, 4, 8):
        raise ValueError(f"batch width must be 1, 2, 4, or 8, got {batch_width}")
    return apply_cost_bitwise(s, plan, gamma)
