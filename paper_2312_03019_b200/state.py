"""Device-resident state vectors.

Mirrors the reference's state module (pkg/src/qaoa_maxcut/state.py): a
``StateVector`` with ``n`` and ``amps`` (complex128, bit i of the index =
qubit i, state.py:3-4), the memory guard ``check_qubit_budget``
(state.py:55-63), single-qubit ``apply_rx`` (state.py:110-128) and the parity
metric ``max_abs_diff`` (state.py:152-156).

Here the amplitudes live in HBM inside an engine context (C ABI
``qaoa_create``).  ``.amps`` materializes a host copy on demand (a
device-to-host read); the host copy then becomes authoritative -- it may be
mutated like the reference's numpy array -- and is uploaded again before the
next engine operation.  Kernels update the state in place and return the same
object, as in the reference (state.py:6-9).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib

DEFAULT_MAX_QUBITS = 26  # state.py:21


def check_qubit_budget(n: int, max_qubits: int = DEFAULT_MAX_QUBITS) -> None:
    """Refuse n above the guard, naming the GiB it would take (state.py:55-63)."""
    if n < 1:
        raise ValueError("qubit count must be at least 1")
    if n > max_qubits:
        gib = 16 * (1 << n) / 2**30
        raise ValueError(
            f"{n} qubits need {gib:.1f} GiB of amplitudes "
            f"(guard is {max_qubits} qubits; raise max_qubits to override)"
        )


class _WriteCounter:
    """Amplitude writes (state.py:27-40): one fused level adds (n+1)*2^n, the
    reference's definition of "amplitude updates"."""

    def __init__(self) -> None:
        self.amp_writes = 0

    def add(self, k: int) -> None:
        self.amp_writes += k

    def reset(self) -> None:
        self.amp_writes = 0


write_counter = _WriteCounter()


class Engine:
    """One engine context (C ABI ``qaoa_ctx``): 2^n complex128 amplitudes in HBM."""

    def __init__(self, n: int, device: int = 0, stream: int | None = None,
                 external_ptr: int | None = None):
        L = _lib.load()
        out = ctypes.c_void_p()
        if external_ptr is None:
            _lib.check(L.qaoa_create(n, device, stream, ctypes.byref(out)))
        else:
            _lib.check(L.qaoa_create_external(n, device, stream, external_ptr, ctypes.byref(out)))
        self._L = L
        self.ptr = out
        self.n = n
        self.device = device
        self.graph_key = None

    def close(self) -> None:
        if self.ptr:
            self._L.qaoa_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_layout_swap(self, mode: int) -> None:
        """Swapped qubit layout policy of qaoa_run_layers (qaoa_set_layout_swap):
        -1 default (on at N=30-type sizes when a second 16 B x 2^n buffer fits),
        0 never (in place, no second buffer), 1 whenever applicable."""
        self.call("qaoa_set_layout_swap", int(mode))

    def trim(self) -> None:
        """Free the second state buffer and the cut table (qaoa_trim)."""
        self.call("qaoa_trim")

    def call(self, name: str, *args) -> None:
        _lib.check(getattr(self._L, name)(self.ptr, *args))

    def state_ptr(self) -> int:
        return int(self._L.qaoa_state_ptr(self.ptr))

    def set_graph(self, g, x_hi: int = 0, row_mask=None, key=None) -> None:
        masks = np.ascontiguousarray(
            np.array(row_mask if row_mask is not None else g.row_mask, dtype=np.uint64))
        self.call("qaoa_set_graph", int(g.n), masks.ctypes.data_as(_lib._u64p), int(g.tot_edge),
                  int(x_hi))
        self.graph_key = key if key is not None else (g.n, tuple(g.row_mask), x_hi)

    def ensure_graph(self, g, x_hi: int = 0) -> None:
        key = (g.n, tuple(g.row_mask), x_hi)
        if self.graph_key != key:
            self.set_graph(g, x_hi, key=key)

    def ensure_weights(self, g) -> None:
        """Weighted edge list on the device (qaoa_set_weights), in Graph.edges order."""
        key = ("w", g.n, tuple(g.edges))
        if getattr(self, "_wkey", None) == key:
            return
        ei = np.ascontiguousarray(np.array([e[0] for e in g.edges], dtype=np.int32))
        ej = np.ascontiguousarray(np.array([e[1] for e in g.edges], dtype=np.int32))
        w = np.ascontiguousarray(np.array([e[2] for e in g.edges], dtype=np.float64))
        self.call("qaoa_set_weights", len(g.edges), ei.ctypes.data_as(_lib._ip),
                  ej.ctypes.data_as(_lib._ip), _lib.dptr(w))
        self._wkey = key

    def write(self, amps: np.ndarray, offset: int = 0) -> None:
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        self.call("qaoa_write_amplitudes", offset, a.size, _lib.dptr(a.view(np.float64)))

    def read(self, offset: int = 0, count: int | None = None) -> np.ndarray:
        count = (1 << self.n) - offset if count is None else count
        out = np.empty(count, dtype=np.complex128)
        self.call("qaoa_read_amplitudes", offset, count, _lib.dptr(out.view(np.float64)))
        return out

    def scalar(self, name: str, *args) -> float:
        out = ctypes.c_double()
        self.call(name, *args, ctypes.byref(out))
        return out.value


class StateVector:
    """n-qubit complex128 state; ``amps`` is the host view (reference state.py:43-52)."""

    __slots__ = ("n", "_host", "_eng", "_where")

    def __init__(self, n: int, amps: np.ndarray | None = None, *, engine: Engine | None = None):
        self.n = int(n)
        self._eng = engine
        if amps is not None:
            a = np.asarray(amps)
            if a.shape != (1 << self.n,):
                raise ValueError(f"amplitude array of shape {a.shape} does not hold {self.n} qubits")
            self._host = a if a.dtype == np.complex128 else a.astype(np.complex128)
            self._where = "host"
        else:
            if engine is None:
                raise ValueError("StateVector needs amplitudes or a device engine")
            self._host = None
            self._where = "device"

    # -- host view ---------------------------------------------------------
    @property
    def amps(self) -> np.ndarray:
        if self._where == "device":
            self._host = self._eng.read()
            self._where = "host"
        return self._host

    @amps.setter
    def amps(self, value: np.ndarray) -> None:
        a = np.asarray(value, dtype=np.complex128)
        if a.shape != (1 << self.n,):
            raise ValueError(f"amplitude array of shape {a.shape} does not hold {self.n} qubits")
        self._host = a
        self._where = "host"

    # -- device view -------------------------------------------------------
    def engine(self, device: int = 0) -> Engine:
        """The device copy, uploaded first if the host copy is authoritative."""
        if self._eng is None:
            self._eng = Engine(self.n, device)
        if self._where == "host":
            self._eng.write(self._host)
            self._where = "device"
            self._host = None
        return self._eng

    @property
    def on_device(self) -> bool:
        return self._where == "device"

    def copy(self) -> "StateVector":
        if self._where == "host":
            return StateVector(self.n, self._host.copy())
        eng = Engine(self.n, self._eng.device)
        src = self._eng.state_ptr()
        _copy_device(eng, src, 16 << self.n)
        return StateVector(self.n, engine=eng)

    def norm(self) -> float:
        """sqrt(sum |a|^2) (state.py:50-51), reduced on the device."""
        return math.sqrt(self.engine().scalar("qaoa_norm_sq"))

    def __repr__(self) -> str:
        return f"StateVector(n={self.n}, where={self._where})"


def _copy_device(dst: Engine, src_ptr: int, nbytes: int) -> None:
    """Device-to-device copy of engine memory (torch's CUDA runtime does the copy)."""
    import torch

    _wrap_device(dst.state_ptr(), nbytes, dst.device).copy_(
        _wrap_device(src_ptr, nbytes, dst.device))
    torch.cuda.synchronize(dst.device)


class _CudaArray:
    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
        }


def _wrap_device(ptr: int, nbytes: int, device: int):
    """Zero-copy torch uint8 view of engine device memory."""
    import torch

    with torch.cuda.device(device):
        return torch.as_tensor(_CudaArray(ptr, nbytes), device=f"cuda:{device}")


def as_tensor(s: StateVector):
    """Zero-copy torch.complex128 view of a device-resident state."""
    import torch

    eng = s.engine()
    t = _wrap_device(eng.state_ptr(), 16 << s.n, eng.device)
    return t.view(torch.complex128)


def init_zero_state(n: int, max_qubits: int = DEFAULT_MAX_QUBITS) -> StateVector:
    """|0...0>: amplitude 1 at index 0 (state.py:66-72), written on the device."""
    check_qubit_budget(n, max_qubits)
    eng = Engine(n)
    eng.call("qaoa_init_basis", 0)
    write_counter.add(1 << n)
    return StateVector(n, engine=eng)


def apply_h(s: StateVector, q: int, threads: int = 1) -> StateVector:
    """Hadamard on qubit q (state.py:91-107): (a +- b) * (1/sqrt 2) with the
    reference's rounding, one device pass."""
    if not 0 <= q < s.n:
        raise IndexError(f"qubit {q} out of range for n={s.n}")
    s.engine().call("qaoa_apply_h", int(q))
    write_counter.add(1 << s.n)
    return s


def rzz_phases(theta: float) -> np.ndarray:
    """(e_same, e_diff) formed exactly as state.py:138-139 forms them."""
    return np.array([complex(np.exp(-0.5j * theta)), complex(np.exp(0.5j * theta))],
                    dtype=np.complex128)


def apply_rzz(s: StateVector, q1: int, q2: int, theta: float, threads: int = 1) -> StateVector:
    """exp(-i theta Z Z / 2) on qubits q1, q2 (state.py:131-149), one device pass,
    bit-exact (numpy's FMA-form complex multiply)."""
    if q1 == q2:
        raise ValueError("RZZ needs two distinct qubits")
    for q in (q1, q2):
        if not 0 <= q < s.n:
            raise IndexError(f"qubit {q} out of range for n={s.n}")
    ph = rzz_phases(theta)
    s.engine().call("qaoa_apply_rzz", int(q1), int(q2), _lib.dptr(ph.view(np.float64)))
    write_counter.add(1 << s.n)
    return s


def apply_rx(s: StateVector, q: int, theta: float, threads: int = 1) -> StateVector:
    """exp(-i theta X / 2) on qubit q (state.py:110-128), bit-exact, on the device."""
    if not 0 <= q < s.n:
        raise IndexError(f"qubit {q} out of range for n={s.n}")
    s.engine().call("qaoa_apply_rx", int(q), math.cos(theta / 2.0), math.sin(theta / 2.0))
    write_counter.add(1 << s.n)
    return s


def max_abs_diff(a: StateVector, b: StateVector) -> float:
    """max_x |a_x - b_x|, no global-phase quotient (state.py:152-156)."""
    if a.n != b.n:
        raise ValueError(f"qubit counts differ: {a.n} vs {b.n}")
    ha, hb = getattr(a, "half_engine", None), getattr(b, "half_engine", None)
    if ha is not None and hb is not None:  # two symmetric halves: their mirrors agree too
        out = ctypes.c_double()
        _lib.check(_lib.load().qaoa_max_abs_diff(ha.ptr, hb.ptr, ctypes.byref(out)))
        return out.value
    if ha is not None or hb is not None:
        return float(np.max(np.abs(a.amps - b.amps)))
    if a.on_device and b.on_device:
        out = ctypes.c_double()
        _lib.check(_lib.load().qaoa_max_abs_diff(a._eng.ptr, b._eng.ptr, ctypes.byref(out)))
        return out.value
    return float(np.max(np.abs(a.amps - b.amps)))


def dump_state(s: StateVector) -> str:
    """One "index real imag" line per amplitude (state.py:159-162)."""
    return "".join(f"{k} {float(v.real)!r} {float(v.imag)!r}\n" for k, v in enumerate(s.amps))
