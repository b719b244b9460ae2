"""ORACLE -- test infrastructure only.

CPU restatements of the reference's RNS-Winograd layer path used to check the
GPU product: ``ref_port`` (numpy, follows rw/layer.py step by step) and the C
direct-convolution oracle in ``oracle.c`` (built into ``oracle/_build``).
Only tests/, __graft_entry__.smoke() and bench.py's CPU baseline / reference
arm may import this package.  The product (paper_2007_12216_b200) never does.
"""

from __future__ import annotations

import ctypes
import os
import shutil
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD = HERE / "_build"
LIB = BUILD / "liboracle.so"

_lib = None


def build(force: bool = False) -> Path:
    """Compile oracle.c -> oracle/_build/liboracle.so (gcc, pthreads)."""
    src = HERE / "oracle.c"
    BUILD.mkdir(exist_ok=True)
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        cc = os.environ.get("CC") or shutil.which("gcc") or "cc"
        subprocess.run([cc, "-O3", "-march=x86-64-v2", "-pthread", "-fPIC", "-shared", str(src), "-o", str(LIB)],
                       check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = ctypes.CDLL(os.fspath(LIB))
        vp, ci = ctypes.c_void_p, ctypes.c_int
        _lib.oracle_direct_conv.restype = ci
        _lib.oracle_direct_conv.argtypes = [vp, vp, ci, ci, ci, ci, ci, ci, ci, vp]
        _lib.oracle_sandwich_mod.restype = None
        _lib.oracle_sandwich_mod.argtypes = [vp, vp, vp, ci, ci, ci, ci, ctypes.c_int32, vp]
        _lib.oracle_mrc.restype = ctypes.c_int64
        _lib.oracle_mrc.argtypes = [vp, vp, ci]
    return _lib


def direct_conv_c(x: np.ndarray, w: np.ndarray, pad: int) -> np.ndarray:
    """Exact int32 conv, NHWC x and (R,R,C,K) w (rw/layer.py:93-103), in C."""
    x = np.ascontiguousarray(x, dtype=np.int8)
    w = np.ascontiguousarray(w, dtype=np.int8)
    b, h, wd, c = x.shape
    r, k = w.shape[0], w.shape[3]
    y = np.empty((b, h + 2 * pad - r + 1, wd + 2 * pad - r + 1, k), dtype=np.int32)
    rc = lib().oracle_direct_conv(x.ctypes.data, w.ctypes.data, b, h, wd, c, k, r, pad, y.ctypes.data)
    if rc:
        raise ValueError(f"oracle_direct_conv failed ({rc})")
    return y
