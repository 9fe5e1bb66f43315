"""Multi-GPU QAOA: the 2^N state sharded over G = 2^g devices by its top g
physical qubits (the reference has no distributed state,
SPEC.md:186).  Rank r holds physical indices [r 2^(N-g), (r+1) 2^(N-g)).

The product path is ``simulate_sharded_fused``: every shard runs the planned
fast schedule of its N-g local qubits in segments (``qaoa_run_begin`` /
``qaoa_run_segment``), and once per level, right after the low set S_0
(local bits 0..11), ONE in-place exchange pass swaps the g global bits with
S_0's top g bits (chunk d of rank r <-> chunk r of rank d, (G-1)/G of each
shard over the links) and applies that level's RX to the qubits that just
became local (``qaoa_exchange`` kernel over peer pointers).  Exchangers:
``IpcExchanger`` (one GPU per process, peers mapped with CUDA IPC, host
barriers), ``IpcChunkExchanger`` (the same, pipelined chunk by chunk with
inter-process CUDA events so the exchange overlaps the sweeps around it),
``PeerExchanger`` / ``PeerChunkExchanger`` (G virtual shards on one device,
for tests).

``simulate_sharded`` is the unfused reference schedule (one engine run per
level, then an all-to-all through ``DistExchanger`` -- torch.distributed P2P,
NCCL on GPUs, gloo on CPU -- or ``LocalExchanger``, then one RX sweep over the
arrived qubits); the tests also drive it with a CPU shard built on the oracle.

Either way the permutation is kept (never swapped back): ``ShardLayout.phys``
tracks the physical bit of every logical qubit, the cost kernels receive the
graph's row masks relabelled to physical positions plus the shard's fixed high
bits, and the fast-mode complement mask is permuted with the data.  <C> is the
fixed-rank-order sum of the shard partials (deterministic).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Protocol, Sequence

import numpy as np

from .circuit import QaoaParams, level_arrays
from .graph import Graph


# --------------------------------------------------------------------------
# qubit placement
# --------------------------------------------------------------------------
@dataclass
class ShardLayout:
    """Logical -> physical qubit placement of a state sharded 2^g ways."""

    n_total: int
    g: int
    phys: list[int] = field(default_factory=list)

    def __post_init__(self):
        if not self.phys:
            self.phys = list(range(self.n_total))
        if self.g < 0 or self.g >= self.n_total:
            raise ValueError("shard bits must be in [0, n)")

    @property
    def n_local(self) -> int:
        return self.n_total - self.g

    def swap_top(self) -> None:
        """Global physical bits n_local+k <-> local physical bits n_local-g+k."""
        nl, g = self.n_local, self.g
        where = {p: q for q, p in enumerate(self.phys)}
        for k in range(g):
            a, b = nl - g + k, nl + k
            qa, qb = where[a], where[b]
            self.phys[qa], self.phys[qb] = b, a
            where[a], where[b] = qb, qa

    def swap_bits(self, x: int, p0: int | None = None) -> int:
        """Apply the same bit swap (local bits p0.. <-> global bits; default the
        top local bits) to a physical index / mask."""
        nl, g = self.n_local, self.g
        p0 = nl - g if p0 is None else p0
        lo = (x >> p0) & ((1 << g) - 1)
        hi = (x >> nl) & ((1 << g) - 1)
        x &= ~((((1 << g) - 1) << p0) | (((1 << g) - 1) << nl))
        return x | (hi << p0) | (lo << nl)

    def swap_at(self, p0: int) -> None:
        """Global physical bits n_local+k <-> local physical bits p0+k."""
        nl, g = self.n_local, self.g
        where = {p: q for q, p in enumerate(self.phys)}
        for k in range(g):
            a, b = p0 + k, nl + k
            qa, qb = where[a], where[b]
            self.phys[qa], self.phys[qb] = b, a
            where[a], where[b] = qb, qa

    def physical_row_masks(self, g: Graph) -> list[int]:
        """Row masks of the graph relabelled to physical bit positions."""
        masks = [0] * self.n_total
        for i, j, _ in g.edges:
            a, b = self.phys[i], self.phys[j]
            if a > b:
                a, b = b, a
            masks[a] |= 1 << b
        return masks

    def logical_to_physical(self, idx: np.ndarray) -> np.ndarray:
        out = np.zeros_like(idx)
        for q, p in enumerate(self.phys):
            out |= ((idx >> np.uint64(q)) & np.uint64(1)) << np.uint64(p)
        return out


# --------------------------------------------------------------------------
# shard engines
# --------------------------------------------------------------------------
class Shard(Protocol):
    rank: int
    n: int

    def set_graph(self, n_nodes: int, masks: Sequence[int], tot_edge: int, x_hi: int) -> None: ...
    def run_level(self, table: np.ndarray, c: float, s: float, first: bool) -> None: ...
    def apply_rx_range(self, q0: int, count: int, c: float, s: float) -> None: ...
    def get_cmask(self) -> int: ...
    def set_cmask(self, m: int) -> None: ...
    def expectation(self) -> float: ...
    def tensor(self): ...
    def synchronize(self) -> None: ...


class CudaShard:
    """One engine context (C ABI) holding one shard on one GPU."""

    def __init__(self, n_local: int, rank: int, device: int = 0, exact: bool = False,
                 stream: int | None = None):
        from . import _lib
        from .state import Engine

        self._lib = _lib
        self.rank = rank
        self.n = n_local
        self.device = device
        self.exact = exact
        if stream is None:  # a stream this side knows, so exchanges can be ordered on it
            import torch

            self._stream = torch.cuda.Stream(device)
            stream = self._stream.cuda_stream
        self.stream_ptr = stream
        self.eng = Engine(n_local, device, stream=stream)

    def set_graph(self, n_nodes, masks, tot_edge, x_hi):
        from . import _lib

        m = np.ascontiguousarray(np.array(masks, dtype=np.uint64))
        self.eng.call("qaoa_set_graph", int(n_nodes), m.ctypes.data_as(_lib._u64p), int(tot_edge),
                      int(x_hi))

    def run_level(self, table, c, s, first):
        from . import _lib

        t = np.ascontiguousarray(table, dtype=np.complex128)
        cs = np.array([c], dtype=np.float64)
        ss = np.array([s], dtype=np.float64)
        flags = (0 if first else _lib.RUN_FROM_STATE) | (_lib.RUN_EXACT if self.exact else 0)
        self.eng.call("qaoa_run_layers", 1, _lib.dptr(t.view(np.float64)), _lib.dptr(cs),
                      _lib.dptr(ss), flags)

    def apply_rx_range(self, q0, count, c, s):
        from . import _lib

        self.eng.call("qaoa_apply_rx_range", int(q0), int(count), float(c), float(s),
                      _lib.RUN_EXACT if self.exact else 0)

    def get_cmask(self) -> int:
        import ctypes

        out = ctypes.c_uint64()
        self.eng.call("qaoa_get_cmask", ctypes.byref(out))
        return int(out.value)

    def set_cmask(self, m: int) -> None:
        self.eng.call("qaoa_set_cmask", int(m))

    def expectation(self) -> float:
        return self.eng.scalar("qaoa_expectation")

    def tensor(self):
        from .state import _wrap_device
        import torch

        return _wrap_device(self.eng.state_ptr(), 16 << self.n, self.device).view(torch.complex128)

    def synchronize(self):
        self.eng.call("qaoa_synchronize")

    # ---- planned runs in segments + fused exchange (the product path) ----------
    def run_begin(self, tables, cs, ss, flags: int) -> int:
        from . import _lib

        self._keep = (np.ascontiguousarray(tables, dtype=np.complex128),
                      np.ascontiguousarray(cs, dtype=np.float64),
                      np.ascontiguousarray(ss, dtype=np.float64))
        t, c, s = self._keep
        nseg = ctypes.c_int()
        self.eng.call("qaoa_run_begin", len(c), _lib.dptr(t.view(np.float64)), _lib.dptr(c),
                      _lib.dptr(s), int(flags), ctypes.byref(nseg))
        return nseg.value

    def run_segment(self, k: int) -> None:
        self.eng.call("qaoa_run_segment", int(k))

    def exchange_info(self, k: int):
        """(level, rx[3], factor[2]) of the exchange after segment k, or None."""
        from . import _lib

        lvl = ctypes.c_int()
        rx = np.zeros(3)
        fac = np.zeros(2)
        rc = self._lib.load().qaoa_run_exchange_info(self.eng.ptr, int(k), ctypes.byref(lvl),
                                                     _lib.dptr(rx), _lib.dptr(fac))
        if rc == _lib.QAOA_E_RANGE:
            return None
        _lib.check(rc)
        return lvl.value, rx, fac

    def run_end(self) -> None:
        self.eng.call("qaoa_run_end")

    def sweep_info(self, i: int):
        """(segment, carry, q, ntiles) of plan sweep i, or None past the end."""
        from . import _lib

        seg, carry, q = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        nt = ctypes.c_int64()
        rc = self._lib.load().qaoa_run_sweep_info(self.eng.ptr, int(i), ctypes.byref(seg),
                                                  ctypes.byref(carry), ctypes.byref(q),
                                                  ctypes.byref(nt))
        if rc == _lib.QAOA_E_RANGE:
            return None
        _lib.check(rc)
        return seg.value, carry.value, q.value, nt.value

    def run_sweep_range(self, i: int, lo: int, count: int) -> None:
        self.eng.call("qaoa_run_sweep_range", int(i), int(lo), int(count))

    @property
    def stream(self):
        """The torch stream the engine launches on (created by this shard)."""
        return self._stream

    def state_ptr(self) -> int:
        return self.eng.state_ptr()

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        self.eng.call("qaoa_ipc_handle", buf)
        return buf.raw

    def close(self):
        self.eng.close()


# --------------------------------------------------------------------------
# exchangers: swap chunk d of shard r with chunk r of shard d (all r != d)
# --------------------------------------------------------------------------
class LocalExchanger:
    """All shards live in this process (virtual shards): pairwise chunk swaps."""

    def __init__(self, shards: Sequence[Shard]):
        self.shards = list(shards)

    def exchange(self, g: int) -> None:
        import torch

        G = len(self.shards)
        ts = [s.tensor() for s in self.shards]
        chunk = ts[0].numel() // G
        for s in self.shards:
            s.synchronize()
        for r in range(G):
            for d in range(r + 1, G):
                a = ts[r][d * chunk:(d + 1) * chunk]
                b = ts[d][r * chunk:(r + 1) * chunk]
                tmp = a.clone()
                a.copy_(b)
                b.copy_(tmp)
        if ts[0].is_cuda:
            torch.cuda.synchronize(ts[0].device)


class DistExchanger:
    """One shard per process; torch.distributed point-to-point in pieces of
    ``piece_elems`` amplitudes through a staging buffer (the in-place swap needs
    no second shard-sized buffer: a 128 GiB shard at N=36, G=8 leaves no room)."""

    def __init__(self, shard: Shard, rank: int, world: int, piece_elems: int = 1 << 24,
                 group=None):
        self.shard = shard
        self.rank = rank
        self.world = world
        self.piece = piece_elems
        self.group = group
        self.staging = None

    def exchange(self, g: int) -> None:
        import torch
        import torch.distributed as dist

        G, r = self.world, self.rank
        dev = torch.view_as_real(self.shard.tensor())  # [2^n, 2] float64 (NCCL has no c128)
        # gloo moves host tensors only: stage device shards through host memory
        host_staged = dev.is_cuda and dist.get_backend(self.group) == "gloo"
        chunk = dev.shape[0] // G
        piece = min(self.piece, chunk)
        peers = [d for d in range(G) if d != r]
        sdev = torch.device("cpu") if host_staged else dev.device
        if self.staging is None or self.staging.shape[0] < piece * len(peers) or \
                self.staging.device != sdev:
            self.staging = torch.empty((piece * len(peers), 2), dtype=dev.dtype, device=sdev)
            self.sendbuf = torch.empty_like(self.staging) if host_staged else None
        self.shard.synchronize()
        for off in range(0, chunk, piece):
            ln = min(piece, chunk - off)
            ops = []
            for k, d in enumerate(peers):
                src = dev[d * chunk + off: d * chunk + off + ln]
                if host_staged:
                    self.sendbuf[k * piece: k * piece + ln].copy_(src)
                    src = self.sendbuf[k * piece: k * piece + ln]
                ops.append(dist.P2POp(dist.isend, src, d, group=self.group))
                ops.append(dist.P2POp(dist.irecv, self.staging[k * piece: k * piece + ln], d,
                                      group=self.group))
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            for k, d in enumerate(peers):
                dev[d * chunk + off: d * chunk + off + ln].copy_(self.staging[k * piece: k * piece + ln])
        if dev.is_cuda:
            torch.cuda.synchronize(dev.device)


# --------------------------------------------------------------------------
# the sharded circuit
# --------------------------------------------------------------------------
def simulate_sharded(g: Graph, params: QaoaParams, shards: Sequence[Shard], exchanger,
                     g_bits: int, layout: ShardLayout | None = None) -> ShardLayout:
    """Run the p-level circuit on a state sharded 2^g_bits ways.  ``shards`` are
    the shards owned by this process (all G for virtual shards, one per rank
    under torch.distributed).  Returns the final qubit layout."""
    n_total = g.n
    layout = layout or ShardLayout(n_total, g_bits)
    nl = layout.n_local
    if g_bits > 9 or nl - g_bits < 0:
        raise ValueError("unsupported shard count")
    tables, cs, ss = level_arrays(g, params)

    def push_graph():
        masks = layout.physical_row_masks(g)
        for sh in shards:
            sh.set_graph(n_total, masks, g.tot_edge, sh.rank << nl)

    push_graph()
    for lvl in range(params.p):
        for sh in shards:
            sh.run_level(tables[lvl], float(cs[lvl]), float(ss[lvl]), first=(lvl == 0))
        if g_bits == 0:
            continue
        exchanger.exchange(g_bits)
        for sh in shards:
            sh.set_cmask(layout.swap_bits(sh.get_cmask()))
        layout.swap_top()
        push_graph()
        for sh in shards:
            sh.apply_rx_range(nl - g_bits, g_bits, float(cs[lvl]), float(ss[lvl]))
    return layout


def sharded_expectation(shards: Sequence[Shard], world_sum=None) -> float:
    """Deterministic <C>: shard partials summed in rank order."""
    parts = {sh.rank: sh.expectation() for sh in shards}
    if world_sum is not None:
        parts = world_sum(parts)
    return float(sum(parts[r] for r in sorted(parts)))


def gather_true_state(layout: ShardLayout, stored: np.ndarray, cmask: int) -> np.ndarray:
    """Host reassembly for tests: stored = concatenation of the shards in rank
    order (physical index = rank << n_local | local).  Returns the state in
    logical order: true[X] = stored[phys(X) ^ cmask]."""
    idx = np.arange(stored.size, dtype=np.uint64)
    return stored[layout.logical_to_physical(idx) ^ np.uint64(cmask)]


# --------------------------------------------------------------------------
# the fused path: segmented shard runs + in-place exchange kernel over peer
# pointers (qaoa_exchange), RX of the arriving qubits fused into the exchange
# --------------------------------------------------------------------------
def exchange_p0(g_bits: int) -> int:
    """Local bits swapped with the global ones: the top g bits of the low set
    S_0 (local bits 0..11), which every level finishes before its exchange."""
    return 12 - g_bits


def _exchange_call(device, stream, g_bits, ptrs, n_local, p0, y_lo, y_hi, rx, factor):
    from . import _lib

    arr = (ctypes.c_void_p * len(ptrs))(*[ctypes.c_void_p(int(p)) for p in ptrs])
    rx = np.ascontiguousarray(rx, dtype=np.float64)
    factor = np.ascontiguousarray(factor, dtype=np.float64)
    _lib.check(_lib.load().qaoa_exchange(int(device), ctypes.c_void_p(stream), int(g_bits), arr,
                                         int(n_local), int(p0), int(y_lo), int(y_hi),
                                         _lib.dptr(rx), _lib.dptr(factor)))


class PeerExchanger:
    """All G shards in this process on one device (virtual shards): one launch
    of the exchange kernel over the G buffers."""

    def __init__(self, shards: Sequence[CudaShard]):
        self.shards = list(shards)
        self.ptrs = [s.state_ptr() for s in self.shards]

    def exchange(self, g_bits: int, p0: int, rx, factor) -> None:
        for s in self.shards:
            s.synchronize()
        import torch

        s0 = self.shards[0]
        _exchange_call(s0.device, s0.stream_ptr, g_bits, self.ptrs, s0.n, p0, 0,
                       1 << (s0.n - g_bits), rx, factor)
        torch.cuda.synchronize(s0.device)


class PeerChunkExchanger(PeerExchanger):
    """Virtual shards in one process, pipelined: exchange chunk t runs on its own
    high-priority stream as soon as every shard's chunk t of the preceding sweep
    is done (stream events, no host waits), and each shard's following sweep on
    chunk t waits only for that exchange chunk."""

    def __init__(self, shards, n_chunks: int):
        import torch

        super().__init__(shards)
        self.n_chunks = n_chunks
        dev = self.shards[0].device
        self.xstream = torch.cuda.Stream(dev, priority=-1)
        c = n_chunks
        self.ev_pre = [[torch.cuda.Event() for _ in range(c)] for _ in self.shards]
        self.ev_x = [torch.cuda.Event() for _ in range(c)]

    # the three phases of one pipelined exchange (see simulate_sharded_fused)
    def after_pre_chunk(self, t: int) -> None:
        for r, sh in enumerate(self.shards):
            self.ev_pre[r][t].record(sh.stream)

    def sync_point(self) -> None:
        pass

    def launch_chunks(self, g_bits, p0, rx, factor) -> None:
        s0 = self.shards[0]
        cols = 1 << (s0.n - g_bits)
        c = self.n_chunks
        for t in range(c):
            for r in range(len(self.shards)):
                self.xstream.wait_event(self.ev_pre[r][t])
            _exchange_call(s0.device, self.xstream.cuda_stream, g_bits, self.ptrs, s0.n, p0,
                           cols * t // c, cols * (t + 1) // c, rx, factor)
            self.ev_x[t].record(self.xstream)

    def wait_chunk(self, shard_index: int, t: int) -> None:
        self.shards[shard_index].stream.wait_event(self.ev_x[t])


class IpcExchanger:
    """One shard per process (one GPU each): the peers' state buffers are mapped
    with CUDA IPC, rank r runs the exchange kernel on its 1/G of the columns with
    P2P loads / stores over NVLink; host barriers order it against the shards'
    sweeps."""

    def __init__(self, shard: CudaShard, rank: int, world: int, group=None):
        import torch.distributed as dist

        from . import _lib

        self.shard, self.rank, self.world, self.group = shard, rank, world, group
        self.timing = False  # set True to time every exchange kernel (CUDA events)
        self._pending: list = []  # per exchange: its (start, stop) event pairs
        self.exchange_ms: list[float] = []  # kernel time per exchange, this rank's slice
        handles = [None] * world
        dist.all_gather_object(handles, shard.ipc_handle(), group=group)
        self.ptrs, self.opened = [], []
        for r, h in enumerate(handles):
            if r == rank:
                self.ptrs.append(shard.state_ptr())
                continue
            out = ctypes.c_void_p()
            buf = ctypes.create_string_buffer(h, 64)
            _lib.check(_lib.load().qaoa_ipc_open(buf, int(shard.device), ctypes.byref(out)))
            self.ptrs.append(out.value)
            self.opened.append(out.value)

    def _barrier(self):
        import torch.distributed as dist

        dist.barrier(group=self.group)

    def exchange(self, g_bits: int, p0: int, rx, factor) -> None:
        sh = self.shard
        cols = 1 << (sh.n - g_bits)
        lo = cols * self.rank // self.world
        hi = cols * (self.rank + 1) // self.world
        sh.synchronize()
        self._barrier()  # every shard finished the segment before anyone reads it
        import torch

        self._begin_exchange()
        ev = self._mark(sh.stream)
        _exchange_call(sh.device, sh.stream_ptr, g_bits, self.ptrs, sh.n, p0, lo, hi, rx, factor)
        self._mark_end(ev, sh.stream)
        torch.cuda.synchronize(sh.device)
        self.collect()
        self._barrier()  # every write into my shard landed before my next sweep

    # ---- per-exchange kernel timing (CUDA events on the launching stream) -----
    def _begin_exchange(self):
        if self.timing:
            self._pending.append([])

    def _mark(self, stream):
        if not self.timing:
            return None
        import torch

        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def _mark_end(self, start, stream):
        if start is None:
            return
        import torch

        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        self._pending[-1].append((start, e))

    def collect(self) -> None:
        """Resolve the timed exchanges (call once their streams have synchronised):
        one entry per exchange = the sum of its kernel launches' durations."""
        for pairs in self._pending:
            self.exchange_ms.append(sum(a.elapsed_time(b) for a, b in pairs))
        self._pending = []

    def close(self) -> None:
        from . import _lib

        for p in self.opened:
            _lib.load().qaoa_ipc_close(ctypes.c_void_p(p))
        self.opened = []


class IpcChunkExchanger(IpcExchanger):
    """One shard per process, pipelined with inter-process CUDA events: rank r's
    exchange stream waits for EVERY rank's chunk-t event of the preceding sweep
    before its slice of exchange chunk t, and its sweep stream waits for every
    rank's exchange-chunk-t event before the following sweep's chunk t.  Two
    host barriers per exchange (over a gloo group: no device synchronisation)
    order the event records before the waits."""

    def __init__(self, shard: CudaShard, rank: int, world: int, n_chunks: int, group=None,
                 ipc_events: bool | None = None):
        import os

        import torch
        import torch.distributed as dist

        super().__init__(shard, rank, world, group)
        self.n_chunks = n_chunks
        self.cpu_group = dist.new_group(backend="gloo")
        if ipc_events is None:  # QAOA_IPC_EVENTS=0: host barriers per chunk instead
            ipc_events = os.environ.get("QAOA_IPC_EVENTS", "1") != "0"
        self.ipc_events = ipc_events
        dev = shard.device
        self.xstream = torch.cuda.Stream(dev, priority=-1)
        mk = lambda: torch.cuda.Event(interprocess=ipc_events, enable_timing=False)  # noqa: E731
        self.my_pre = [mk() for _ in range(n_chunks)]
        self.my_x = [mk() for _ in range(n_chunks)]
        if not ipc_events:
            return
        # events must exist on the device before their IPC handles are taken
        with torch.cuda.stream(shard.stream):
            for e in self.my_pre + self.my_x:
                e.record()
        torch.cuda.synchronize(dev)
        mine = ([e.ipc_handle() for e in self.my_pre], [e.ipc_handle() for e in self.my_x])
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=self.cpu_group)
        self.pre = [[self.my_pre[t] if r == rank else torch.cuda.Event.from_ipc_handle(dev, allh[r][0][t])
                     for t in range(n_chunks)] for r in range(world)]
        self.x = [[self.my_x[t] if r == rank else torch.cuda.Event.from_ipc_handle(dev, allh[r][1][t])
                   for t in range(n_chunks)] for r in range(world)]

    def after_pre_chunk(self, t: int) -> None:
        self.my_pre[t].record(self.shard.stream)

    def _host_barrier(self) -> None:
        import torch.distributed as dist

        dist.barrier(group=self.cpu_group)

    def sync_point(self) -> None:
        if self.ipc_events:
            self._host_barrier()

    def launch_chunks(self, g_bits, p0, rx, factor) -> None:
        sh = self.shard
        cols = 1 << (sh.n - g_bits)
        c, G, r = self.n_chunks, self.world, self.rank
        self._begin_exchange()
        for t in range(c):
            if self.ipc_events:
                for rr in range(G):
                    self.xstream.wait_event(self.pre[rr][t])
            else:  # every rank's chunk t of the sweep is done
                self.my_pre[t].synchronize()
                self._host_barrier()
            lo, hi = cols * t // c, cols * (t + 1) // c
            ev = self._mark(self.xstream)  # after the waits: the chunk's kernel time only
            _exchange_call(sh.device, self.xstream.cuda_stream, g_bits, self.ptrs, sh.n, p0,
                           lo + (hi - lo) * r // G, lo + (hi - lo) * (r + 1) // G, rx, factor)
            self._mark_end(ev, self.xstream)
            self.my_x[t].record(self.xstream)

    def wait_chunk(self, shard_index: int, t: int) -> None:
        if self.ipc_events:
            for rr in range(self.world):
                self.shard.stream.wait_event(self.x[rr][t])
        else:  # every rank's exchange chunk t landed
            self.my_x[t].synchronize()
            self._host_barrier()


def simulate_sharded_fused(g: Graph, params: QaoaParams, shards: Sequence[CudaShard], exchanger,
                           g_bits: int, exact: bool = False, expect: bool = False,
                           timing: bool = False, layout: ShardLayout | None = None) -> ShardLayout:
    """p levels on a state sharded 2^g_bits ways with the fused schedule: per
    level the shard-local sweeps of the fast plan (level-boundary sweeps merged
    as on one GPU) stop once after the low set S_0 for ONE exchange that swaps
    the global qubits with S_0's top g bits and applies this level's RX to the
    arriving ones (R - 1 local sweeps + 1 exchange pass per level for R local
    qubit sets).  ``shards`` are those owned by this process."""
    from . import _lib

    n_total = g.n
    layout = layout or ShardLayout(n_total, g_bits)
    nl = layout.n_local
    if g_bits < 1 or g_bits > 4 or nl < 12:
        raise ValueError("fused sharding needs 1..4 shard bits and >= 12 local qubits")
    p0 = exchange_p0(g_bits)
    tables, cs, ss = level_arrays(g, params)

    def push_graph():
        masks = layout.physical_row_masks(g)
        for sh in shards:
            sh.set_graph(n_total, masks, g.tot_edge, sh.rank << nl)

    push_graph()
    pipelined = getattr(exchanger, "n_chunks", 1) > 1
    flags = _lib.RUN_SHARDED | (_lib.RUN_EXACT if exact else 0) | \
        (_lib.RUN_EXPECTATION if expect else 0) | \
        (_lib.RUN_TIMING if timing and not pipelined else 0)
    nseg = [sh.run_begin(tables, cs, ss, flags) for sh in shards][0]

    def relabel():
        for sh in shards:
            sh.set_cmask(layout.swap_bits(sh.get_cmask(), p0))
        layout.swap_at(p0)
        push_graph()

    if not pipelined:
        for k in range(nseg):
            for sh in shards:
                sh.run_segment(k)
            info = shards[0].exchange_info(k)
            if info is None:
                continue
            _, rx, factor = info
            exchanger.exchange(g_bits, p0, rx, factor)
            relabel()
    else:
        _run_pipelined(shards, exchanger, nseg, g_bits, p0, nl, relabel)
    for sh in shards:
        sh.run_end()
    return layout


def _run_pipelined(shards, exchanger, nseg, g_bits, p0, nl, relabel):
    """Exchange k overlapped with the sweeps around it, chunk by chunk: the chunk
    of a tile is its top log2(C) local index bits, so every sweep whose qubits
    avoid those bits splits into C contiguous tile ranges.  The sweep before
    the exchange (S_0) runs chunk by chunk and signals each chunk; exchange
    chunk t runs (own stream) once every shard's chunk t is done; the sweep
    after the exchange (when its qubits avoid the chunk bits) runs chunk t once
    exchange chunk t is done everywhere.  Everything else runs whole."""
    C = exchanger.n_chunks
    cb = C.bit_length() - 1
    sweeps = []
    i = 0
    while True:
        info = shards[0].sweep_info(i)
        if info is None:
            break
        sweeps.append(info)
        i += 1
    by_seg = [[j for j, s in enumerate(sweeps) if s[0] == k] for k in range(nseg)]

    def chunkable(j):
        _, carry, q, _ = sweeps[j]
        top = 11 if carry >= 12 else q + 11 - carry  # highest qubit the sweep mixes
        return top < nl - cb

    def ranges(j):
        nt = sweeps[j][3]
        return [(nt * t // C, nt * (t + 1) // C - nt * t // C) for t in range(C)]

    skip_first = False
    for k in range(nseg):
        js = by_seg[k]
        ex = shards[0].exchange_info(k)
        pre = js[-1] if ex is not None else None
        body = js[1:] if skip_first else js
        if pre is not None:
            body = body[:-1] if body and body[-1] == pre else body
        for j in body:
            for sh in shards:
                sh.run_sweep_range(j, 0, sweeps[j][3])
        if ex is None:
            skip_first = False
            continue
        _, rx, factor = ex
        # the sweep before the exchange, chunk by chunk (whole when it cannot split)
        if chunkable(pre):
            for t, (lo, cnt) in enumerate(ranges(pre)):
                for sh in shards:
                    sh.run_sweep_range(pre, lo, cnt)
                exchanger.after_pre_chunk(t)
        else:
            for sh in shards:
                sh.run_sweep_range(pre, 0, sweeps[pre][3])
            for t in range(C):
                exchanger.after_pre_chunk(t)
        exchanger.sync_point()
        exchanger.launch_chunks(g_bits, p0, rx, factor)
        exchanger.sync_point()
        relabel()  # the following sweeps see the swapped layout
        nxt = by_seg[k + 1][0] if k + 1 < nseg and by_seg[k + 1] else None
        # (a one-sweep segment followed by an exchange runs its sweep as that
        # exchange's pre-sweep instead)
        nxt_is_pre = nxt is not None and len(by_seg[k + 1]) == 1 and \
            shards[0].exchange_info(k + 1) is not None
        if nxt is not None and chunkable(nxt) and not nxt_is_pre:
            for t, (lo, cnt) in enumerate(ranges(nxt)):
                for r, sh in enumerate(shards):
                    exchanger.wait_chunk(r, t)
                    sh.run_sweep_range(nxt, lo, cnt)
            skip_first = True
        else:
            for t in range(C):
                for r, sh in enumerate(shards):
                    exchanger.wait_chunk(r, t)
            skip_first = False
