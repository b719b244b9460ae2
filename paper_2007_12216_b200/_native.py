"""ctypes binding of the C ABI in include/rnsw.h (librnsw.so, built in-tree).

There is no fallback: if the shared object is missing or fails to load the
import raises, so a GPU box can never silently run a CPU path.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import raise_for

_PRODUCT_LIB = Path(__file__).resolve().parent / "librnsw.so"


def _lib_path() -> Path:
    """The in-tree librnsw.so.  Diagnostic A/B builds (tools/ab_*.sh, some of
    which skip loads or MMAs and compute wrong answers on purpose) load only
    when RNSW_DIAG=1 is set together with RNSW_LIB, and announce themselves on
    stderr; bench.py records the override in its JSON line."""
    override = os.environ.get("RNSW_LIB")
    if override and os.environ.get("RNSW_DIAG") == "1":
        import sys

        print(f"[rnsw] DIAGNOSTIC library {override} (RNSW_DIAG=1): results may be wrong by design",
              file=sys.stderr)
        return Path(override)
    return _PRODUCT_LIB


_LIB_PATH = _lib_path()
_lock = threading.Lock()
_lib = None

c_int, c_int64, c_size_t, c_void_p = ctypes.c_int, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p
_i8p = ctypes.POINTER(ctypes.c_int8)
_i16p = ctypes.POINTER(ctypes.c_int16)
_i32p = ctypes.POINTER(ctypes.c_int32)

# name -> (restype, argtypes)
_SIGNATURES = {
    "rnsw_plan_create": (c_int, [ctypes.POINTER(c_void_p), c_int, c_int, c_int, _i32p, _i16p, _i16p, _i16p, _i32p]),
    "rnsw_plan_destroy": (None, [c_void_p]),
    "rnsw_plan_info": (c_int, [c_void_p, ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
    "rnsw_filter_bytes": (c_size_t, [c_void_p, c_int, c_int]),
    "rnsw_v_bytes": (c_size_t, [c_void_p, c_int64, c_int]),
    "rnsw_m_bytes": (c_size_t, [c_void_p, c_int64, c_int]),
    "rnsw_workspace_bytes": (c_size_t, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int]),
    "rnsw_filter_transform": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, c_size_t, c_void_p]),
    "rnsw_filter_import": (c_int, [c_void_p, c_int, c_void_p, c_int, c_int, c_void_p, c_size_t, c_void_p]),
    "rnsw_input_transform": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                     c_size_t, c_void_p]),
    "rnsw_input_transform_compact": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int,
                                             c_void_p, c_size_t, c_void_p]),
    "rnsw_small_channel_product": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p,
                                           c_size_t, c_void_p]),
    "rnsw_winograd_gemm": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p, c_size_t,
                                   c_void_p]),
    "rnsw_output_transform": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                      c_void_p]),
    "rnsw_output_residues": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_void_p]),
    "rnsw_conv_forward": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                  c_void_p, c_void_p, c_size_t, c_void_p]),
    "rnsw_conv_forward_timed": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                        c_void_p, c_void_p, c_void_p, c_size_t, c_void_p,
                                        ctypes.POINTER(ctypes.c_float)]),
    "rnsw_conv_forward_ev": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                     c_void_p, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    "rnsw_conv_forward_requant_ev": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                             c_int, c_int, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    "rnsw_tile_decompose": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_size_t,
                                    c_void_p]),
    "rnsw_conv_forward_requant": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                          c_int, c_int, c_void_p, c_void_p, c_size_t, c_void_p]),
    "rnsw_output_transform_requant": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                              c_void_p, c_void_p]),
    "rnsw_mw8_supported": (c_int, [c_void_p]),
    "rnsw_small_channel_product_mw8": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p,
                                               c_size_t, c_void_p]),
    "rnsw_winograd_gemm_mw8": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p, c_size_t,
                                       c_void_p]),
    "rnsw_output_transform_mw8": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                          c_void_p]),
    "rnsw_output_transform_requant_mw8": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int,
                                                  c_int, c_void_p, c_void_p]),
    "rnsw_direct_weight_bytes": (c_size_t, [c_int, c_int, c_int]),
    "rnsw_direct_pack_weights": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_size_t, c_void_p]),
    "rnsw_direct_conv": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_int, c_int, c_int, c_int,
                                 c_void_p, c_void_p]),
    "rnsw_mrc_reconstruct": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "rnsw_requant_pool": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p]),
    "rnsw_error_string": (ctypes.c_char_p, [c_int]),
    "rnsw_last_error": (ctypes.c_char_p, []),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

LAYOUT_NHWC = 0
LAYOUT_NCHW = 1


def library_path() -> Path:
    return _LIB_PATH


def lib():
    """Load librnsw.so once (raises if it is absent: no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise ImportError(
                    f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(the RNS-Winograd path has no CPU fallback)"
                )
            handle = ctypes.CDLL(os.fspath(_LIB_PATH))
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


RNSW_OK = 0


def check(rc: int) -> None:
    if rc != 0:
        l = lib()
        raise_for(rc, f"{l.rnsw_error_string(rc).decode()}: {l.rnsw_last_error().decode()}")


class Plan:
    """Owns one ``rnsw_plan*`` (constant tables for one (tile, R, moduli))."""

    def __init__(self, tile_m: int, r: int, moduli, at: np.ndarray, g: np.ndarray, bt: np.ndarray,
                 mrc_inv: np.ndarray):
        l = lib()
        self.tile_m, self.r = int(tile_m), int(r)
        self.moduli = tuple(int(m) for m in moduli)
        mods = np.ascontiguousarray(self.moduli, dtype=np.int32)
        at = np.ascontiguousarray(at, dtype=np.int16)
        g = np.ascontiguousarray(g, dtype=np.int16)
        bt = np.ascontiguousarray(bt, dtype=np.int16)
        inv = np.ascontiguousarray(mrc_inv, dtype=np.int32)
        # identity of the modular transform matrices: two plans with the same
        # key compute the same filter bank (default and custom points differ)
        import hashlib

        self.key = (self.tile_m, self.r, self.moduli,
                    hashlib.sha1(at.tobytes() + g.tobytes() + bt.tobytes()).hexdigest())
        handle = c_void_p()
        check(l.rnsw_plan_create(ctypes.byref(handle), self.tile_m, self.r, len(self.moduli),
                                 mods.ctypes.data_as(_i32p), at.ctypes.data_as(_i16p), g.ctypes.data_as(_i16p),
                                 bt.ctypes.data_as(_i16p), inv.ctypes.data_as(_i32p)))
        self._h = handle
        n, planes = c_int(), c_int()
        check(l.rnsw_plan_info(handle, ctypes.byref(n), ctypes.byref(planes)))
        self.n, self.n_planes = n.value, planes.value

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.rnsw_plan_destroy(h)
            self._h = None
