"""The C ABI library loads on a CPU-only host and exports exactly what
include/rnsw.h declares (no compute calls without a GPU)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2007_12216_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    text = (ROOT / "include" / "rnsw.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rnsw_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    for name in declared_functions():
        assert getattr(lib, name) is not None, name
    assert Path(_native.library_path()).name.startswith("librnsw")


def test_error_strings_without_device():
    lib = _native.lib()
    assert lib.rnsw_error_string(0) == b"ok"
    assert lib.rnsw_error_string(4) == b"dynamic range exceeded"
    assert lib.rnsw_error_string(99) == b"unknown error"


def test_plan_validation_rejects_bad_arguments_before_device_work():
    import numpy as np

    lib = _native.lib()
    h = ctypes.c_void_p()
    mods = np.array([6, 7], dtype=np.int32)
    z16 = np.zeros(1024, dtype=np.int16)
    inv = np.zeros(4, dtype=np.int32)
    i16 = ctypes.POINTER(ctypes.c_int16)
    i32 = ctypes.POINTER(ctypes.c_int32)
    rc = lib.rnsw_plan_create(ctypes.byref(h), 4, 3, 2, mods.ctypes.data_as(i32), z16.ctypes.data_as(i16),
                              z16.ctypes.data_as(i16), z16.ctypes.data_as(i16), inv.ctypes.data_as(i32))
    assert rc == 1  # even modulus -> RNSW_ERR_INVALID
    mods = np.array([21, 35], dtype=np.int32)
    rc = lib.rnsw_plan_create(ctypes.byref(h), 4, 3, 2, mods.ctypes.data_as(i32), z16.ctypes.data_as(i16),
                              z16.ctypes.data_as(i16), z16.ctypes.data_as(i16), inv.ctypes.data_as(i32))
    assert rc == 5  # share factor 7 -> RNSW_ERR_NOT_COPRIME
    rc = lib.rnsw_plan_create(ctypes.byref(h), 23, 3, 1, mods.ctypes.data_as(i32), z16.ctypes.data_as(i16),
                              z16.ctypes.data_as(i16), z16.ctypes.data_as(i16), inv.ctypes.data_as(i32))
    assert rc == 10  # N = 25 > 24 -> RNSW_ERR_UNSUPPORTED
    assert b"exceeds" in lib.rnsw_last_error()


def test_sources_target_sm100a_only():
    from paper_2007_12216_b200 import build

    flags = " ".join(build.NVCC_FLAGS)
    assert "arch=compute_100a,code=sm_100a" in flags
    assert "sm_90" not in flags and "compute_90" not in flags
    for src in build.sources():
        text = src.read_text()
        assert "wgmma" not in text and "triton" not in text.lower()
