"""The drop-in boundary: libqaoa_b200.so loads (no GPU needed) and exports
every entry point include/qaoa_b200.h declares, with the ctypes binding of the
Python package covering exactly that set."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2312_03019_b200 import _lib


@pytest.fixture(scope="module")
def lib_path():
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    return _lib.LIB_PATH


def header_functions():
    text = open(_lib.HEADER).read()
    return sorted(set(re.findall(r"QAOA_API\s+[\w\s\*]*?\b(qaoa_\w+)\s*\(", text)))


def test_header_parsed():
    names = header_functions()
    assert "qaoa_run_layers" in names and "qaoa_expectation" in names
    assert len(names) >= 25


def test_library_exports_header(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True)
    exported = set(re.findall(r"\bT (qaoa_\w+)", out.stdout))
    missing = [n for n in header_functions() if n not in exported]
    assert not missing, missing
    # nothing but the C ABI leaks out of the library
    assert exported == set(header_functions())


def test_binding_matches_header():
    assert sorted(_lib.SIGNATURES) == header_functions()


def test_loads_without_gpu(lib_path):
    L = _lib.load()
    assert L.qaoa_version().decode().startswith("qaoa_b200")
    n = L.qaoa_device_count()
    assert n >= 0
    if n == 0:
        out = ctypes.c_void_p()
        rc = L.qaoa_create(10, 0, None, ctypes.byref(out))
        assert rc == _lib.QAOA_E_CUDA
        assert "CUDA" in _lib.last_error()


def test_error_mapping():
    with pytest.raises(ValueError):
        _lib.check(_lib.QAOA_E_INVALID)
    with pytest.raises(IndexError):
        _lib.check(_lib.QAOA_E_RANGE)
    with pytest.raises(MemoryError):
        _lib.check(_lib.QAOA_E_NOMEM)
    with pytest.raises(_lib.EngineError):
        _lib.check(_lib.QAOA_E_CUDA)
