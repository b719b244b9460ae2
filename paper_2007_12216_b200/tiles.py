"""Single-tile API of the reference (rw/kernel.py:56-105) on the device.

``tile_conv_mod`` (one modulus) and ``rns_tile_conv`` (all residues + MRC)
are public in the reference but not on the layer path.  Here every tile pair
runs as a one-tile layer through the same kernels as ``winograd_layer_conv``
(H = W = N, C = K = 1, no padding), so the tile API and the layer path share
one implementation.  Tile pairs are batched per distinct filter.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from .errors import DynamicRangeExceeded, ShapeMismatch
from .layer import LayerSpec, winograd_layer_conv
from .residue import RnsSystem
from .transforms import ModularTransformSet, cached_transforms, reduce_transforms_mod


def _torch():
    import torch

    return torch


def _check_set(mt: ModularTransformSet) -> None:
    """The device derives its tables from cached_transforms(m, r); a caller's
    set must be that one (rw/kernel.py takes any set, the device path only
    the default points)."""
    ref = reduce_transforms_mod(cached_transforms(mt.m, mt.r), mt.modulus)
    if not (np.array_equal(ref.at, mt.at) and np.array_equal(ref.g, mt.g) and np.array_equal(ref.bt, mt.bt)):
        raise ShapeMismatch(f"transform set for F({mt.m},{mt.r}) mod {mt.modulus} is not the default-points set; "
                            "the device path only has those")


def _pairs(g, d, r: int, n: int):
    """Broadcast (..., r, r) filters against (..., n, n) tiles -> flat stacks."""
    g = np.asarray(g)
    d = np.asarray(d)
    if g.shape[-2:] != (r, r):
        raise ShapeMismatch(f"filter tile must be {r}x{r}, got {g.shape[-2:]}")
    if d.shape[-2:] != (n, n):
        raise ShapeMismatch(f"input tile must be {n}x{n}, got {d.shape[-2:]}")
    lead = np.broadcast_shapes(g.shape[:-2], d.shape[:-2])
    gs = np.broadcast_to(g, lead + (r, r)).reshape(-1, r, r)
    ds = np.broadcast_to(d, lead + (n, n)).reshape(-1, n, n)
    return lead, gs, ds


def _tile_layer(gs: np.ndarray, ds: np.ndarray, m_out: int, r: int, system: RnsSystem, declared_bound):
    """(S, r, r) x (S, n, n) int8 -> (S, m, m) int32 on the device: one layer
    call (batch = tiles) per distinct filter."""
    torch = _torch()
    n = m_out + r - 1
    s = gs.shape[0]
    out = torch.empty((s, m_out, m_out), dtype=torch.int32, device="cuda")
    if s == 0:
        return out
    uniq, inv = np.unique(gs.reshape(s, r * r), axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    x_all = torch.from_numpy(np.ascontiguousarray(ds, dtype=np.int8)).cuda()
    for u in range(uniq.shape[0]):
        idx = np.nonzero(inv == u)[0]
        sel = torch.from_numpy(idx).cuda()
        spec = LayerSpec(h=n, w=n, c=1, k=1, r=r, padding=0, batch=len(idx), tile_m=m_out)
        w = torch.from_numpy(uniq[u].reshape(r, r, 1, 1).astype(np.int8)).cuda()
        y = winograd_layer_conv(spec, w, x_all.index_select(0, sel).unsqueeze(-1).contiguous(), system,
                                declared_bound=declared_bound)
        out.index_copy_(0, sel, y[..., 0])
    return out


def _int8_tiles(a: np.ndarray, what: str) -> np.ndarray:
    if a.size and (a.min() < -128 or a.max() > 127):
        raise ValueError(f"{what} must be in the int8 range for the device path")
    return a.astype(np.int8)


def tile_conv_mod(g, d, mt: ModularTransformSet) -> np.ndarray:
    """One fast correlation tile modulo one modulus (rw/kernel.py:56-70).

    g: (..., r, r) filter residues, d: (..., n, n) input residues; returns the
    (..., m, m) symmetric output residues, congruent to the direct
    correlation.  16-bit moduli: residues are split into s8 limbs
    (v = 256 hi + lo) and the four limb products are recombined mod m.
    """
    torch = _torch()
    _check_set(mt)
    m, r, n = mt.modulus, mt.r, mt.m + mt.r - 1
    lead, gs, ds = _pairs(g, d, r, n)
    half = (m - 1) // 2
    gs = ((gs.astype(np.int64) + half) % m - half)
    ds = ((ds.astype(np.int64) + half) % m - half)
    system = RnsSystem((m,))
    if m < 256:
        y = _tile_layer(gs.astype(np.int8), ds.astype(np.int8), mt.m, r, system, 0)
    else:
        def limbs(v):
            lo = (v + 128) % 256 - 128
            return lo.astype(np.int8), ((v - lo) // 256).astype(np.int8)

        g_lo, g_hi = limbs(gs)
        d_lo, d_hi = limbs(ds)
        t = {(a, b): _tile_layer(ga, db, mt.m, r, system, 0).to(torch.int64)
             for a, ga in ((0, g_lo), (1, g_hi)) for b, db in ((0, d_lo), (1, d_hi))}
        acc = t[0, 0] + 256 * (t[0, 1] + t[1, 0]) + 65536 * t[1, 1]
        y = torch.remainder(acc + half, m) - half
    return y.to(torch.int32).cpu().numpy().reshape(lead + (mt.m, mt.m))


def rns_tile_conv(g, d, system: RnsSystem, mts: Sequence[ModularTransformSet]) -> np.ndarray:
    """One full-precision tile: every residue, then mixed-radix reconstruction
    (rw/kernel.py:73-105).  Same checks in the same order: ShapeMismatch for
    a transform-set list that does not match the system, then
    DynamicRangeExceeded when r*r*127^2 exceeds the signed bound."""
    if len(mts) != len(system.moduli):
        raise ShapeMismatch(f"expected {len(system.moduli)} transform sets, got {len(mts)}")
    for mt, m in zip(mts, system.moduli):
        if mt.modulus != m:
            raise ShapeMismatch(f"transform set for modulus {mt.modulus} does not match system {system}")
    r = mts[0].r
    worst = r * r * 127 * 127
    if worst > system.signed_bound:
        raise DynamicRangeExceeded(f"worst case output {worst} exceeds signed bound {system.signed_bound}")
    for mt in mts:
        _check_set(mt)
    m_out = mts[0].m
    lead, gs, ds = _pairs(g, d, r, m_out + r - 1)
    y = _tile_layer(_int8_tiles(gs, "filter tiles"), _int8_tiles(ds, "input tiles"), m_out, r, system, None)
    return y.cpu().numpy().reshape(lead + (m_out, m_out))
