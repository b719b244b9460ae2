"""Residue number systems: symmetric residues, inverses, MRC constants.

Host-side restatement of the array half of rw/residue.py.  Residues live in
the symmetric range [-(m-1)/2, (m-1)/2] of an odd modulus m (rw/residue.py:
25-33), moduli are capped at 15 bits so residues fit int16 (rw/residue.py:16),
and reconstruction is mixed-radix conversion with the inverse table
``mrc_inv[j][i] = m_i^-1 mod m_j`` for i < j (rw/residue.py:70-81).  The
device kernels receive that table through the plan (include/rnsw.h); nothing
here touches tensor data.
"""

from __future__ import annotations

import math
from typing import Sequence

import numpy as np

from .errors import NotCoprime, OutOfRange, SystemMismatch

MAX_MODULUS = (1 << 15) - 1


def check_modulus(m) -> int:
    """Accept odd integers in [3, 2**15 - 1] (rw/residue.py:19-24)."""
    if isinstance(m, bool) or not isinstance(m, (int, np.integer)):
        raise TypeError(f"modulus must be an integer, got {type(m).__name__}")
    if m < 3 or m % 2 == 0 or m > MAX_MODULUS:
        raise ValueError(f"modulus must be odd and in [3, {MAX_MODULUS}], got {m}")
    return int(m)


def mod_reduce(x: int, m: int) -> int:
    """Symmetric residue of x modulo m (rw/residue.py:27-33)."""
    check_modulus(m)
    r = x % m
    return r - m if r > (m - 1) // 2 else r


def mod_inverse(x: int, m: int) -> int:
    """Symmetric inverse of x modulo m; NotCoprime when none exists."""
    check_modulus(m)
    try:
        inv = pow(int(x), -1, m)
    except ValueError:
        raise NotCoprime(f"{x} is not invertible modulo {m}") from None
    return mod_reduce(inv, m)


class RnsSystem:
    """Pairwise-coprime odd moduli plus the constants the device MRC needs.

    Immutable and hashable like the reference class (rw/residue.py:56-92).
    """

    def __init__(self, moduli: Sequence[int]):
        mods = tuple(check_modulus(m) for m in moduli)
        if not mods:
            raise ValueError("an RNS system needs at least one modulus")
        for i, a in enumerate(mods):
            for b in mods[i + 1 :]:
                g = math.gcd(a, b)
                if g != 1:
                    raise NotCoprime(f"moduli {a} and {b} share factor {g}")
        self.moduli = mods
        self.dynamic_range = math.prod(mods)
        self.signed_bound = (self.dynamic_range - 1) // 2
        # mrc_inv[j][i] = m_i^-1 mod m_j (i < j), symmetric representative
        self._mrc_inv = [[mod_inverse(mods[i], mods[j]) for i in range(j)] for j in range(len(mods))]

    def __len__(self) -> int:
        return len(self.moduli)

    def __eq__(self, other) -> bool:
        return isinstance(other, RnsSystem) and self.moduli == other.moduli

    def __hash__(self) -> int:
        return hash(self.moduli)

    def __repr__(self) -> str:
        return f"RnsSystem{self.moduli}"

    def mrc_table(self) -> np.ndarray:
        """Dense (n, n) int32 table T[j][i] = m_i^-1 mod m_j for i < j, else 0."""
        n = len(self.moduli)
        t = np.zeros((n, n), dtype=np.int32)
        for j in range(n):
            for i in range(j):
                t[j, i] = self._mrc_inv[j][i]
        return t

    def encode(self, x: int) -> tuple[int, ...]:
        """Scalar encode (host convenience; the layer path never calls it)."""
        if abs(x) > self.signed_bound:
            raise OutOfRange(f"{x} outside representable range +/-{self.signed_bound}")
        return tuple(mod_reduce(x, m) for m in self.moduli)

    def reconstruct(self, residues) -> int:
        """Scalar mixed-radix reconstruction into the signed range."""
        vals = tuple(residues)
        if len(vals) != len(self.moduli):
            raise SystemMismatch(f"expected {len(self.moduli)} residues, got {len(vals)}")
        digits: list[int] = []
        for j, m in enumerate(self.moduli):
            t = vals[j] % m
            for i in range(j):
                t = (t - digits[i]) * self._mrc_inv[j][i] % m
            digits.append(t)
        x = 0
        for j in range(len(digits) - 1, -1, -1):
            x = x * self.moduli[j] + digits[j]
        return x - self.dynamic_range if x > self.signed_bound else x


def planes_for_modulus(m: int) -> int:
    """int8 limb planes one residue occupies on the tensor cores.

    m < 256: residues fit s8 -> 1 plane.  Otherwise the residue v is split as
    v = 256*hi + lo with lo the sign-extended low byte and hi in [-64, 64],
    both s8 -> 2 planes (the int16 storage of rw/gemm.py:25-27, re-expressed
    for ``tcgen05.mma.kind::i8``).
    """
    return 1 if m < 256 else 2
