"""ctypes binding of the C ABI in include/qaoa_b200.h (libqaoa_b200.so).

The shared library is built in-tree (paper_2312_03019_b200/_lib/) by
``python -c "import __graft_entry__ as g; g.build()"`` or ``make -C
paper_2312_03019_b200/csrc``.  There is no fallback: if the library or a GPU
is missing, every engine call raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "_lib")
LIB_PATH = os.environ.get("QAOA_B200_LIB") or os.path.join(LIB_DIR, "libqaoa_b200.so")
CSRC = os.path.join(_HERE, "csrc")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "qaoa_b200.h")

QAOA_OK = 0
QAOA_E_INVALID = -1
QAOA_E_RANGE = -2
QAOA_E_CUDA = -3
QAOA_E_NOMEM = -4
QAOA_E_STATE = -5

RUN_EXACT = 0x1
RUN_FROM_STATE = 0x2
RUN_EXPECTATION = 0x4
RUN_TIMING = 0x8
RUN_SHARDED = 0x10
RUN_EXPECT_ONLY = 0x20
RUN_MIRROR = 0x40

_c_int = ctypes.c_int
_c_dbl = ctypes.c_double
_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_ip = ctypes.POINTER(ctypes.c_int)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)

# name -> (restype, argtypes); mirrors include/qaoa_b200.h
SIGNATURES = {
    "qaoa_last_error": (ctypes.c_char_p, []),
    "qaoa_version": (ctypes.c_char_p, []),
    "qaoa_device_count": (_c_int, []),
    "qaoa_create": (_c_int, [_c_int, _c_int, _vp, ctypes.POINTER(_vp)]),
    "qaoa_create_external": (_c_int, [_c_int, _c_int, _vp, _vp, ctypes.POINTER(_vp)]),
    "qaoa_destroy": (None, [_vp]),
    "qaoa_state_ptr": (_vp, [_vp]),
    "qaoa_set_stream": (_c_int, [_vp, _vp]),
    "qaoa_set_graph": (_c_int, [_vp, _c_int, _u64p, _c_int, _u64]),
    "qaoa_init_uniform": (_c_int, [_vp]),
    "qaoa_write_amplitudes": (_c_int, [_vp, _u64, _u64, _dp]),
    "qaoa_read_amplitudes": (_c_int, [_vp, _u64, _u64, _dp]),
    "qaoa_apply_cost": (_c_int, [_vp, _dp]),
    "qaoa_apply_rx": (_c_int, [_vp, _c_int, _c_dbl, _c_dbl]),
    "qaoa_apply_mixer": (_c_int, [_vp, _c_dbl, _c_dbl]),
    "qaoa_init_basis": (_c_int, [_vp, _u64]),
    "qaoa_apply_h": (_c_int, [_vp, _c_int]),
    "qaoa_apply_rzz": (_c_int, [_vp, _c_int, _c_int, _dp]),
    "qaoa_edge_values": (_c_int, [_vp, _c_int, _u64, _u64, _dp]),
    "qaoa_mirror_rx": (_c_int, [_vp, _dp, _dp]),
    "qaoa_run_layers": (_c_int, [_vp, _c_int, _dp, _dp, _dp, _c_int]),
    "qaoa_apply_rx_range": (_c_int, [_vp, _c_int, _c_int, _c_dbl, _c_dbl, _c_int]),
    "qaoa_set_layout_swap": (_c_int, [_vp, _c_int]),
    "qaoa_set_mirror": (_c_int, [_vp, _c_int]),
    "qaoa_trim": (_c_int, [_vp]),
    "qaoa_get_cmask": (_c_int, [_vp, _u64p]),
    "qaoa_set_cmask": (_c_int, [_vp, _u64]),
    "qaoa_expectation": (_c_int, [_vp, _dp]),
    "qaoa_set_weights": (_c_int, [_vp, _c_int, _ip, _ip, _dp]),
    "qaoa_apply_cost_weighted": (_c_int, [_vp, _c_dbl]),
    "qaoa_expectation_weighted": (_c_int, [_vp, _dp]),
    "qaoa_norm_sq": (_c_int, [_vp, _dp]),
    "qaoa_block_norms": (_c_int, [_vp, _c_int, _dp]),
    "qaoa_sample_blocks": (_c_int, [_vp, _c_int, ctypes.c_int64, _i64p, _dp, _i64p, _dp, _i64p]),
    "qaoa_max_abs_diff": (_c_int, [_vp, _vp, _dp]),
    "qaoa_build_cut_table": (_c_int, [_vp]),
    "qaoa_read_cut_table": (_c_int, [_vp, _u64, _u64, _i64p]),
    "qaoa_free_cut_table": (_c_int, [_vp]),
    "qaoa_layer_timings": (_c_int, [_vp, _fp, _c_int]),
    "qaoa_last_run_stats": (_c_int, [_vp, _ip, _dp]),
    "qaoa_synchronize": (_c_int, [_vp]),
    "qaoa_pack_chunks": (_c_int, [_vp, _c_int, _ip, _vp]),
    "qaoa_unpack_chunks": (_c_int, [_vp, _c_int, _ip, _vp]),
    "qaoa_run_layers_weighted": (_c_int, [_vp, _c_int, _dp, _dp, _dp, _c_int]),
    "qaoa_plan": (_c_int, [_c_int, _c_int, _c_int, _ip, _c_int]),
    "qaoa_run_begin": (_c_int, [_vp, _c_int, _dp, _dp, _dp, _c_int, _ip]),
    "qaoa_run_segment": (_c_int, [_vp, _c_int]),
    "qaoa_run_exchange_info": (_c_int, [_vp, _c_int, _ip, _dp, _dp]),
    "qaoa_run_end": (_c_int, [_vp]),
    "qaoa_run_sweep_info": (_c_int, [_vp, _c_int, _ip, _ip, _ip, _i64p]),
    "qaoa_run_sweep_range": (_c_int, [_vp, _c_int, ctypes.c_int64, ctypes.c_int64]),
    "qaoa_exchange": (_c_int, [_c_int, _vp, _c_int, ctypes.POINTER(_vp), _c_int, _c_int, _u64, _u64,
                               _dp, _dp]),
    "qaoa_ipc_handle": (_c_int, [_vp, _vp]),
    "qaoa_ipc_open": (_c_int, [_vp, _c_int, ctypes.POINTER(_vp)]),
    "qaoa_ipc_close": (_c_int, [_vp]),
}

_lib = None
_lock = threading.Lock()


class EngineError(RuntimeError):
    """A CUDA-side failure of the engine (QAOA_E_CUDA / QAOA_E_STATE)."""


def build(verbose: bool = False) -> str:
    """Compile csrc/*.cu for sm_100a into _lib/libqaoa_b200.so (nvcc, see csrc/Makefile)."""
    out = subprocess.run(["make", "-s", "-C", CSRC], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"building libqaoa_b200.so failed:\n{out.stdout}\n{out.stderr}")
    if verbose:
        print(out.stdout, out.stderr)
    return LIB_PATH


def load():
    """Load the engine library (no fallback: raises if it is not built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: the CUDA engine is not built "
                "(run `make -C paper_2312_03019_b200/csrc` or __graft_entry__.build())"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("QAOA_B200_LIB") and not hasattr(lib, name):
                continue  # A/B tooling: an older build may lack newer entry points
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().qaoa_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    """Map a QAOA_E* status onto the reference's exception types."""
    if rc == QAOA_OK:
        return
    msg = last_error()
    if rc == QAOA_E_INVALID:
        raise ValueError(msg)
    if rc == QAOA_E_RANGE:
        raise IndexError(msg)
    if rc == QAOA_E_NOMEM:
        raise MemoryError(msg)
    raise EngineError(msg or f"engine error {rc}")


def device_count() -> int:
    return int(load().qaoa_device_count())


def dptr(a):
    return a.ctypes.data_as(_dp)
