"""QTNS tensor files: the reference's on-disk format for int8 / int32 tensors
(rw/layer.py:453-504), used by the CLI's file mode.

Layout (all little endian): b"QTNS", u8 version (1), u8 rank, rank x i32
dims, u8 element width in bits (8 or 32), then the C-order payload.  Host
file I/O only; no arithmetic.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import ShapeMismatch

QTNS_MAGIC = b"QTNS"
QTNS_VERSION = 1
_WIDTHS = {8: np.dtype("int8"), 32: np.dtype("<i4")}


def _host_array(arr) -> np.ndarray:
    if hasattr(arr, "detach"):  # torch tensor, possibly on the device
        arr = arr.detach().cpu().numpy()
    return np.asarray(arr)


def write_tensor(path, arr) -> None:
    """Write an int8 or int32 tensor (numpy array or torch tensor).

    Raises ShapeMismatch for other dtypes or rank > 255 (rw/layer.py:457-468).
    """
    a = _host_array(arr)
    bits = {np.dtype("int8"): 8, np.dtype("int32"): 32}.get(a.dtype)
    if bits is None:
        raise ShapeMismatch(f"only int8/int32 tensors are serialized, got {a.dtype}")
    if a.ndim > 255:
        raise ShapeMismatch("rank too large")
    header = QTNS_MAGIC + struct.pack("<BB", QTNS_VERSION, a.ndim)
    header += struct.pack(f"<{a.ndim}i", *a.shape) + struct.pack("<B", bits)
    with open(path, "wb") as f:
        f.write(header)
        f.write(np.ascontiguousarray(a, dtype=_WIDTHS[bits]).tobytes())


def read_tensor(path) -> np.ndarray:
    """Read a QTNS file back (rw/layer.py:480-504).

    ValueError for a wrong magic, version or element width, or a payload
    whose size does not match the dims.
    """
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:4] != QTNS_MAGIC:
        raise ValueError(f"{path}: not a QTNS tensor file")
    if len(raw) < 6:
        raise ValueError(f"{path}: truncated header")
    version, rank = struct.unpack_from("<BB", raw, 4)
    if version != QTNS_VERSION:
        raise ValueError(f"{path}: unsupported version {version}")
    pos = 6
    if len(raw) < pos + 4 * rank + 1:
        raise ValueError(f"{path}: truncated header")
    dims = struct.unpack_from(f"<{rank}i", raw, pos)
    pos += 4 * rank
    (bits,) = struct.unpack_from("<B", raw, pos)
    pos += 1
    if bits not in _WIDTHS:
        raise ValueError(f"{path}: unsupported element width {bits}")
    dt = _WIDTHS[bits]
    count = 1
    for d in dims:
        count *= d
    if len(raw) - pos != count * dt.itemsize:
        raise ValueError(f"{path}: payload is {len(raw) - pos} bytes, expected {count * dt.itemsize}")
    out = np.frombuffer(raw, dtype=dt, count=count, offset=pos).reshape(dims)
    return out.astype(np.int32) if bits == 32 else out.copy()
