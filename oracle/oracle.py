"""ctypes wrapper over the CPU oracle (oracle/qaoa_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg, never by the product
package.  Each wrapper names the reference function it restates
(paths relative to /root/reference/pkg/src/qaoa_maxcut/).

Parity is pinned against golden vectors made by running the reference itself
(tests/golden/make_golden.py); see tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liborc.so")
_lib = None

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    """Compile the oracle (gcc; see oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_cut_counts.argtypes = [ctypes.c_int, _u64p, _i64p, ctypes.c_int]
        L.orc_init_uniform.argtypes = [ctypes.c_int, _f64p, ctypes.c_int]
        L.orc_apply_cost.argtypes = [ctypes.c_int, _u64p, ctypes.c_int, _f64p, _f64p, ctypes.c_int]
        L.orc_apply_rx.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                   _f64p, ctypes.c_int]
        L.orc_apply_mixer.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, _f64p,
                                      ctypes.c_int]
        L.orc_simulate.argtypes = [ctypes.c_int, _u64p, ctypes.c_int, ctypes.c_int, _f64p, _f64p,
                                   _f64p, _f64p, ctypes.c_int]
        L.orc_expectation.argtypes = [ctypes.c_int, _u64p, _f64p, ctypes.c_int]
        L.orc_expectation.restype = ctypes.c_double
        L.orc_norm.argtypes = [ctypes.c_int, _f64p, ctypes.c_int]
        L.orc_norm.restype = ctypes.c_double
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_apply_h.argtypes = [ctypes.c_int, ctypes.c_int, _f64p, ctypes.c_int]
        L.orc_apply_rzz.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _f64p, _f64p,
                                    ctypes.c_int]
        L.orc_apply_cost_x.argtypes = [ctypes.c_int, ctypes.c_int, _u64p, ctypes.c_uint64,
                                       ctypes.c_int, _f64p, _f64p, ctypes.c_int]
        L.orc_expectation_x.argtypes = [ctypes.c_int, ctypes.c_int, _u64p, ctypes.c_uint64, _f64p,
                                        ctypes.c_int]
        L.orc_expectation_x.restype = ctypes.c_double
        _lib = L
    return _lib


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _masks(row_mask) -> np.ndarray:
    return np.ascontiguousarray(np.array([int(m) for m in row_mask], dtype=np.uint64))


def phase_table(tot_edge: int, gamma: float) -> np.ndarray:
    """cost.py:136-139 (_phase_table), the same numpy expression."""
    levels = np.arange(-tot_edge, tot_edge + 1, dtype=np.float64)
    return np.exp(-0.5j * gamma * levels)


def rx_coeffs(beta: float) -> tuple[float, float]:
    """state.py:114-115 with theta = -beta (circuit.py:93): (cos(theta/2), sin(theta/2))."""
    theta = -beta
    return math.cos(theta / 2.0), math.sin(theta / 2.0)


def max_threads() -> int:
    return int(lib().orc_max_threads())


def cut_counts(n: int, row_mask, threads: int = 0) -> np.ndarray:
    """cost.py:88-99 (CompressedCostPlan.cut_counts)."""
    out = np.empty(1 << n, dtype=np.int64)
    m = _masks(row_mask)
    lib().orc_cut_counts(n, _ptr(m, _u64p), _ptr(out, _i64p), threads)
    return out


def init_uniform(n: int, threads: int = 0) -> np.ndarray:
    """circuit.py:42-48."""
    amps = np.empty(1 << n, dtype=np.complex128)
    lib().orc_init_uniform(n, _ptr(amps, _f64p), threads)
    return amps


def apply_cost(amps: np.ndarray, n: int, row_mask, tot_edge: int, gamma: float,
               threads: int = 0) -> np.ndarray:
    """cost.py:162-176 (apply_cost_bitwise), in place."""
    assert amps.dtype == np.complex128 and amps.flags.c_contiguous
    table = np.ascontiguousarray(phase_table(tot_edge, gamma))
    m = _masks(row_mask)
    lib().orc_apply_cost(n, _ptr(m, _u64p), tot_edge, _ptr(table, _f64p), _ptr(amps, _f64p),
                         threads)
    return amps


def apply_rx(amps: np.ndarray, n: int, q: int, theta: float, threads: int = 0) -> np.ndarray:
    """state.py:110-128, in place."""
    lib().orc_apply_rx(n, q, math.cos(theta / 2.0), math.sin(theta / 2.0), _ptr(amps, _f64p),
                       threads)
    return amps


def apply_h(amps: np.ndarray, n: int, q: int, threads: int = 0) -> np.ndarray:
    """state.py:91-107, in place."""
    lib().orc_apply_h(n, q, _ptr(amps, _f64p), threads)
    return amps


def apply_rzz(amps: np.ndarray, n: int, q1: int, q2: int, theta: float,
              threads: int = 0) -> np.ndarray:
    """state.py:131-149, in place; the two phases formed as the reference forms them."""
    ph = np.array([complex(np.exp(-0.5j * theta)), complex(np.exp(0.5j * theta))],
                  dtype=np.complex128)
    lib().orc_apply_rzz(n, q1, q2, _ptr(ph, _f64p), _ptr(amps, _f64p), threads)
    return amps


def simulate_gates(n: int, edges, gammas, betas, launch_control: bool = True,
                   threads: int = 0) -> np.ndarray:
    """simulate(..., backend="baseline"), circuit.py:97-113: init_state
    (circuit.py:51-62: uniform, or |0..0> plus n Hadamards), then per level one
    RZZ(w gamma) per edge in edge order (circuit.py:76-80) and RX(-beta) per qubit."""
    if launch_control:
        amps = init_uniform(n, threads)
    else:
        amps = np.zeros(1 << n, dtype=np.complex128)
        amps[0] = 1.0
        for q in range(n):
            apply_h(amps, n, q, threads)
    for gm, bt in zip(gammas, betas):
        for e in edges:
            i, j = int(e[0]), int(e[1])
            w = float(e[2]) if len(e) > 2 else 1.0
            apply_rzz(amps, n, i, j, w * gm, threads)
        for q in range(n):
            apply_rx(amps, n, q, -bt, threads)
    return amps


def apply_mixer(amps: np.ndarray, n: int, beta: float, threads: int = 0) -> np.ndarray:
    """circuit.py:89-94, in place."""
    c, s = rx_coeffs(beta)
    lib().orc_apply_mixer(n, c, s, _ptr(amps, _f64p), threads)
    return amps


def simulate(n: int, row_mask, tot_edge: int, gammas, betas, threads: int = 0) -> np.ndarray:
    """circuit.py:97-113 with backend="bitwise", launch_control=True."""
    p = len(gammas)
    tables = np.ascontiguousarray(np.stack([phase_table(tot_edge, g) for g in gammas]))
    cs = np.array([rx_coeffs(b)[0] for b in betas], dtype=np.float64)
    ss = np.array([rx_coeffs(b)[1] for b in betas], dtype=np.float64)
    amps = np.empty(1 << n, dtype=np.complex128)
    m = _masks(row_mask)
    lib().orc_simulate(n, _ptr(m, _u64p), tot_edge, p, _ptr(tables, _f64p), _ptr(cs, _f64p),
                       _ptr(ss, _f64p), _ptr(amps, _f64p), threads)
    return amps


def expectation(n: int, row_mask, amps: np.ndarray, threads: int = 0) -> float:
    """circuit.py:116-121 (unweighted graphs)."""
    m = _masks(row_mask)
    return float(lib().orc_expectation(n, _ptr(m, _u64p), _ptr(amps, _f64p), threads))


def norm(n: int, amps: np.ndarray, threads: int = 0) -> float:
    """state.py:50-51."""
    return float(lib().orc_norm(n, _ptr(amps, _f64p), threads))


def simulate_slice(n_local: int, n_nodes: int, row_mask, x_hi: int, tot_edge: int, gammas, betas,
                   threads: int = 0) -> np.ndarray:
    """The 2^n_local amplitudes of a graph with n_nodes > n_local nodes whose top
    node bits are fixed to x_hi (one shard's index space, no RX on the fixed
    bits): init u = sqrt(1/2^n_nodes) (circuit.py:45), then per level the
    bitwise cost at x_hi | y (cost.py:162-176) and the mixer on the n_local
    qubits (circuit.py:89-94).  Checks the engine's 64-bit-mask path
    (graph.py:41-42 allows N <= 64) on a slice a CPU can hold."""
    a = np.full(1 << n_local, math.sqrt(1.0 / (1 << n_nodes)), dtype=np.complex128)
    m = _masks(row_mask)
    for gm, bt in zip(gammas, betas):
        tab = np.ascontiguousarray(phase_table(tot_edge, gm))
        lib().orc_apply_cost_x(n_local, n_nodes, _ptr(m, _u64p), x_hi, tot_edge, _ptr(tab, _f64p),
                               _ptr(a, _f64p), threads)
        c, s = rx_coeffs(bt)
        lib().orc_apply_mixer(n_local, c, s, _ptr(a, _f64p), threads)
    return a


def expectation_slice(n_local: int, n_nodes: int, row_mask, x_hi: int, amps: np.ndarray,
                      threads: int = 0) -> float:
    """sum_y |a_y|^2 C(x_hi | y) (circuit.py:116-121 restricted to one slice)."""
    m = _masks(row_mask)
    return float(lib().orc_expectation_x(n_local, n_nodes, _ptr(m, _u64p), x_hi,
                                         _ptr(amps, _f64p), threads))


class OracleShard:
    """CPU shard for the sharded-host tests (paper_2312_03019_b200.sharded.Shard
    protocol): reference arithmetic on a numpy shard of global indices x_hi | y."""

    def __init__(self, n_local: int, rank: int, threads: int = 1):
        import torch

        self.rank = rank
        self.n = n_local
        self.threads = threads
        self.t = torch.zeros(1 << n_local, dtype=torch.complex128)
        self.masks = None
        self.n_nodes = 0
        self.tot_edge = 0
        self.x_hi = 0

    def set_graph(self, n_nodes, masks, tot_edge, x_hi):
        self.n_nodes, self.tot_edge, self.x_hi = n_nodes, tot_edge, x_hi
        self.masks = _masks(masks)

    def _amps(self):
        return self.t.numpy()

    def run_level(self, table, c, s, first):
        a = self._amps()
        if first:
            a[:] = math.sqrt(1.0 / (1 << self.n_nodes))
        tab = np.ascontiguousarray(table, dtype=np.complex128)
        lib().orc_apply_cost_x(self.n, self.n_nodes, _ptr(self.masks, _u64p), self.x_hi,
                               self.tot_edge, _ptr(tab, _f64p), _ptr(a, _f64p), self.threads)
        lib().orc_apply_mixer(self.n, c, s, _ptr(a, _f64p), self.threads)

    def apply_rx_range(self, q0, count, c, s):
        a = self._amps()
        for q in range(q0, q0 + count):
            lib().orc_apply_rx(self.n, q, c, s, _ptr(a, _f64p), self.threads)

    def get_cmask(self):
        return 0

    def set_cmask(self, m):
        assert m == 0

    def expectation(self):
        a = self._amps()
        return float(lib().orc_expectation_x(self.n, self.n_nodes, _ptr(self.masks, _u64p),
                                             self.x_hi, _ptr(a, _f64p), self.threads))

    def tensor(self):
        return self.t

    def synchronize(self):
        pass

    # segmented protocol of the fused sharded path (sharded.simulate_sharded_fused):
    # segment k = cost_k + RX_k on every local qubit; the exchange after it
    # applies RX_k (exact form) to the arriving qubits; the last segment is empty.
    def run_begin(self, tables, cs, ss, flags):
        self._run = (np.asarray(tables), np.asarray(cs), np.asarray(ss))
        return len(cs) + 1

    def run_segment(self, k):
        tables, cs, ss = self._run
        if k < len(cs):
            self.run_level(tables[k], float(cs[k]), float(ss[k]), first=(k == 0))

    def exchange_info(self, k):
        tables, cs, ss = self._run
        if k >= len(cs):
            return None
        return k, np.array([cs[k], ss[k], 0.0]), np.array([1.0, 0.0])

    def run_end(self):
        pass

    def state_ptr(self):
        return self


def fused_exchange_numpy(arrays, g, p0, rx):
    """CPU restatement of the fused exchange kernel (qaoa_exchange.cu) on G numpy
    shards in place: element (shard r, local (y, h)) -> (shard h, local (y, r)),
    then the exact RX (c = rx[0], s = rx[1], reference rounding, state.py:114-124)
    on the arriving bits p0.. of every shard, bit by bit in increasing order."""
    G = 1 << g
    n = int(arrays[0].size).bit_length() - 1
    lo = 1 << p0
    mid = 1 << g
    hi = 1 << (n - p0 - g)
    views = [a.reshape(hi, mid, lo) for a in arrays]
    old = [v.copy() for v in views]
    for h in range(G):
        for r in range(G):
            views[h][:, r, :] = old[r][:, h, :]
    c, s = float(rx[0]), float(rx[1])
    for a in arrays:
        for k in range(g):
            lib().orc_apply_rx(n, p0 + k, c, s, _ptr(a, _f64p), 1)


# ---------------------------------------------------------------------------
# Input generators restated from the reference (needed on the GPU box, where
# /root/reference does not exist).  Pinned by tests/test_oracle_golden.py.
# ---------------------------------------------------------------------------

def random_regular_edges(n: int, d: int, seed: int = 0, max_tries: int = 500):
    """graph.py:170-205 (random_regular_graph, unweighted): pairing model."""
    import random

    if d >= n:
        raise ValueError(f"degree {d} must be less than node count {n}")
    if (n * d) % 2 != 0:
        raise ValueError(f"n*d = {n * d} is odd; no {d}-regular graph on {n} nodes")
    rng = random.Random(seed)
    for _ in range(max_tries):
        stubs = [v for v in range(n) for _ in range(d)]
        rng.shuffle(stubs)
        pairs = set()
        ok = True
        for a, b in zip(stubs[::2], stubs[1::2]):
            if a == b:
                ok = False
                break
            e = (min(a, b), max(a, b))
            if e in pairs:
                ok = False
                break
            pairs.add(e)
        if ok:
            return sorted(pairs)
    raise RuntimeError("pairing model failed")


def params_from_seed(p: int, seed: int):
    """bench.py:61-67: gamma in [0, 2pi) drawn first, then beta in [0, pi)."""
    rng = np.random.default_rng(seed)
    gamma = tuple(float(v) for v in rng.uniform(0.0, 2.0 * math.pi, p))
    beta = tuple(float(v) for v in rng.uniform(0.0, math.pi, p))
    return gamma, beta


def row_masks(n: int, edges) -> list[int]:
    """graph.py:57-59: bit j of row_mask[i] set iff edge (i, j), i < j."""
    masks = [0] * n
    for e in edges:
        i, j = int(e[0]), int(e[1])
        if i > j:
            i, j = j, i
        masks[i] |= 1 << j
    return masks


def p1_closed_form(n: int, edges, gamma: float, beta: float) -> float:
    """p=1 per-edge closed form (Wang-Hadfield-Jiang-Rieffel
    mapped to the reference convention).  Reaches sizes the state vector cannot."""
    adj = [set() for _ in range(n)]
    for i, j in edges:
        adj[i].add(j)
        adj[j].add(i)
    s2b = math.sin(2 * beta)
    sb2 = math.sin(beta) ** 2
    cg = math.cos(gamma)
    c2g = math.cos(2 * gamma)
    sg = math.sin(gamma)
    total = 0.0
    for u, v in edges:
        du = len(adj[u]) - 1
        dv = len(adj[v]) - 1
        lam = len(adj[u] & adj[v])
        total += 0.5 + 0.25 * s2b * sg * (cg ** du + cg ** dv) \
            - 0.25 * sb2 * cg ** (du + dv - 2 * lam) * (1 - c2g ** lam)
    return total
