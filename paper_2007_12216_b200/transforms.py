"""Exact Winograd transform construction and its reduction modulo each residue.

Host-side plan construction, restating rw/transforms.py:

* interpolation points 0, 1, -1, 2, -2, ... closed by the point at infinity
  (rw/transforms.py:58-70);
* the Vandermonde inverse in closed form from Lagrange basis polynomials, the
  infinity column holding the coefficients of prod(x - s) over the finite
  points (rw/transforms.py:124-150);
* BT row k = column k of that inverse scaled by the lcm of its denominators,
  G row k = (1, s, ..., s^(r-1)) divided by the same lcm (0,...,0,1 for
  infinity), AT[i][j] = s_j^i with the infinity column e_(m-1)
  (rw/transforms.py:212-238);
* every entry p/q reduced to the symmetric residue p * q^-1 mod m
  (rw/transforms.py:303-331).

All arithmetic is exact (``fractions.Fraction``).  The modular matrices are the
only thing the device needs; they are handed to the native plan as int16.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache
from typing import Sequence

import numpy as np

from . import residue
from .errors import NotCoprime


class _Infinity:
    """Singleton interpolation point at infinity (leading coefficient)."""

    _one = None

    def __new__(cls):
        if cls._one is None:
            cls._one = super().__new__(cls)
        return cls._one

    def __repr__(self) -> str:
        return "INF"


INF = _Infinity()


def default_points(n: int) -> tuple:
    """0, 1, -1, 2, -2, ... (n-1 finite points) followed by INF."""
    if n < 2:
        raise ValueError(f"need at least 2 interpolation points, got {n}")
    finite = [Fraction(0)]
    step = 1
    while len(finite) < n - 1:
        finite.append(Fraction(step))
        if len(finite) < n - 1:
            finite.append(Fraction(-step))
        step += 1
    return tuple(finite) + (INF,)


def _normalise_points(points: Sequence) -> tuple:
    pts = []
    for idx, p in enumerate(points):
        if p is INF:
            if idx != len(points) - 1:
                raise ValueError("the point at infinity must come last")
            pts.append(INF)
        else:
            pts.append(Fraction(p))
    fin = [p for p in pts if p is not INF]
    if len(set(fin)) != len(fin):
        raise ValueError(f"interpolation points must be distinct: {points}")
    return tuple(pts)


def _monic_from_roots(roots: Sequence[Fraction]) -> list[Fraction]:
    """Coefficients, lowest order first, of prod (x - root)."""
    poly = [Fraction(1)]
    for root in roots:
        shifted = [Fraction(0)] + poly  # x * poly
        for i, c in enumerate(poly):
            shifted[i] -= root * c
        poly = shifted
    return poly


def _horner(poly: Sequence[Fraction], x: Fraction) -> Fraction:
    acc = Fraction(0)
    for c in reversed(poly):
        acc = acc * x + c
    return acc


def vandermonde(points: Sequence) -> tuple:
    pts = _normalise_points(points)
    n = len(pts)
    out = []
    for p in pts:
        if p is INF:
            out.append(tuple(Fraction(1 if j == n - 1 else 0) for j in range(n)))
        else:
            out.append(tuple(p**j for j in range(n)))
    return tuple(out)


def vandermonde_inverse(points: Sequence) -> tuple:
    """Closed-form inverse of ``vandermonde(points)`` (no linear solve)."""
    pts = _normalise_points(points)
    n = len(pts)
    has_inf = pts[-1] is INF
    fin = list(pts[:-1]) if has_inf else list(pts)
    inv = [[Fraction(0)] * n for _ in range(n)]
    for j, s in enumerate(fin):
        basis = _monic_from_roots([t for k, t in enumerate(fin) if k != j])
        scale = _horner(basis, s)
        for i, c in enumerate(basis):
            inv[i][j] = c / scale
    if has_inf:
        for i, c in enumerate(_monic_from_roots(fin)):
            inv[i][n - 1] = c
    return tuple(tuple(r) for r in inv)


def _lcm_of_denominators(values) -> int:
    lcm = 1
    for v in values:
        lcm = lcm * v.denominator // math.gcd(lcm, v.denominator)
    return lcm


@dataclass(frozen=True)
class ExactTransformSet:
    """Exact AT (M x N), G (N x R), BT (N x N) for F(M x M, R x R)."""

    m: int
    r: int
    points: tuple
    at: tuple
    g: tuple
    bt: tuple
    alpha: Fraction
    gprime: tuple

    @property
    def n(self) -> int:
        return self.m + self.r - 1


def derive_transforms(m: int, r: int, points: Sequence | None = None) -> ExactTransformSet:
    if m < 1 or r < 1:
        raise ValueError(f"need m >= 1 and r >= 1, got m={m}, r={r}")
    n = m + r - 1
    if n < 2:
        raise ValueError("m + r - 1 must be at least 2")
    pts = default_points(n) if points is None else _normalise_points(points)
    if len(pts) != n:
        raise ValueError(f"need {n} points for m={m}, r={r}, got {len(pts)}")

    vinv = vandermonde_inverse(pts)
    bt, lams = [], []
    for k in range(n):
        col = [vinv[i][k] for i in range(n)]
        lam = _lcm_of_denominators(col)
        lams.append(lam)
        bt.append(tuple(v * lam for v in col))

    g = []
    for k, p in enumerate(pts):
        raw = [Fraction(0)] * (r - 1) + [Fraction(1)] if p is INF else [p**e for e in range(r)]
        g.append(tuple(v / lams[k] for v in raw))

    at = []
    for i in range(m):
        at.append(tuple(Fraction(1 if i == m - 1 else 0) if p is INF else p**i for p in pts))

    alpha = Fraction(1, _lcm_of_denominators(v for row in g for v in row))
    gprime = tuple(tuple(int(v / alpha) for v in row) for row in g)
    return ExactTransformSet(m=m, r=r, points=pts, at=tuple(at), g=tuple(g), bt=tuple(bt),
                             alpha=alpha, gprime=gprime)


@lru_cache(maxsize=64)
def cached_transforms(m: int, r: int) -> ExactTransformSet:
    return derive_transforms(m, r)


def denominator_lcm(ts: ExactTransformSet) -> int:
    return _lcm_of_denominators(v for mat in (ts.g, ts.bt) for row in mat for v in row)


def check_modulus_compatibility(ts: ExactTransformSet, m: int) -> bool:
    """True when every denominator of G and BT is invertible mod m."""
    if isinstance(m, bool) or not isinstance(m, (int, np.integer)) or m < 2:
        raise ValueError(f"modulus must be an integer >= 2, got {m!r}")
    return math.gcd(denominator_lcm(ts), int(m)) == 1


@dataclass(frozen=True)
class ModularTransformSet:
    """The exact set reduced modulo one modulus (int8 if m < 256 else int16)."""

    modulus: int
    at: np.ndarray
    g: np.ndarray
    bt: np.ndarray

    @property
    def m(self) -> int:
        return self.at.shape[0]

    @property
    def r(self) -> int:
        return self.g.shape[1]

    @property
    def n(self) -> int:
        return self.bt.shape[0]


def _reduce_entry(v: Fraction, m: int) -> int:
    if v.denominator == 1:
        return residue.mod_reduce(v.numerator, m)
    return residue.mod_reduce(v.numerator * residue.mod_inverse(v.denominator, m), m)


def _reduce(rows, m: int) -> np.ndarray:
    dt = np.int8 if m < 256 else np.int16
    out = np.array([[_reduce_entry(v, m) for v in row] for row in rows], dtype=dt)
    out.flags.writeable = False
    return out


def reduce_transforms_mod(ts: ExactTransformSet, m: int) -> ModularTransformSet:
    residue.check_modulus(m)
    return ModularTransformSet(modulus=int(m), at=_reduce(ts.at, m), g=_reduce(ts.g, m), bt=_reduce(ts.bt, m))


def reduce_for_system(ts: ExactTransformSet, system: residue.RnsSystem) -> tuple[ModularTransformSet, ...]:
    return tuple(reduce_transforms_mod(ts, m) for m in system.moduli)


__all__ = [
    "INF", "ExactTransformSet", "ModularTransformSet", "NotCoprime",
    "default_points", "vandermonde", "vandermonde_inverse", "derive_transforms",
    "cached_transforms", "denominator_lcm", "check_modulus_compatibility",
    "reduce_transforms_mod", "reduce_for_system",
]
