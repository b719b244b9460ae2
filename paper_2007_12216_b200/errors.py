"""Exception hierarchy of the RNS-Winograd layer path.

Same class names and meaning as the reference package (rw/errors.py:4-33) so
callers that catch ``rnswinograd`` errors keep working after switching.  The
native library reports failures as integer codes (include/rnsw.h); ``raise_for``
maps each code onto one of these classes.
"""

from __future__ import annotations


class RnsError(Exception):
    """Root of every error raised by this package."""


class NotCoprime(RnsError):
    """Two moduli (or a denominator and a modulus) share a factor."""


class SystemMismatch(RnsError):
    """Residues from different RNS systems, or the wrong number of residues."""


class OutOfRange(RnsError):
    """A value does not fit the signed range of the residue system."""


class DynamicRangeExceeded(RnsError):
    """The layer's bound on |output| exceeds the system's signed bound."""


class ShapeMismatch(RnsError):
    """Operand shapes, dtypes or layouts are incompatible."""


class OverflowRisk(RnsError):
    """An int32 accumulator could overflow for the requested reduction length."""


class UnsupportedStride(RnsError):
    """The tiled fast path only handles unit stride."""


class DeviceError(RnsError):
    """The CUDA runtime or the native library failed (not a caller error)."""


# Return codes of the C ABI (include/rnsw.h) -> exception classes.
_CODE_TO_EXC = {
    1: ValueError,  # RNSW_ERR_INVALID
    2: ShapeMismatch,  # RNSW_ERR_SHAPE
    3: UnsupportedStride,  # RNSW_ERR_STRIDE
    4: DynamicRangeExceeded,  # RNSW_ERR_RANGE
    5: NotCoprime,  # RNSW_ERR_NOT_COPRIME
    6: OverflowRisk,  # RNSW_ERR_OVERFLOW
    7: SystemMismatch,  # RNSW_ERR_SYSTEM
    8: DeviceError,  # RNSW_ERR_CUDA
    9: ValueError,  # RNSW_ERR_WORKSPACE
    10: DeviceError,  # RNSW_ERR_UNSUPPORTED
}


def raise_for(code: int, message: str) -> None:
    """Raise the exception class that corresponds to a native return code."""
    if code == 0:
        return
    raise _CODE_TO_EXC.get(code, DeviceError)(message)
