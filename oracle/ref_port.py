"""ORACLE -- test infrastructure only, never shipped or measured as the product.

A CPU restatement (numpy) of the reference's layer-level RNS-Winograd path,
``rnswinograd.layer.winograd_layer_conv`` (rw/layer.py:301-389), and of its
exact oracle ``direct_conv`` (rw/layer.py:81-103).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import this module.

Parity is pinned: tests/test_oracle.py checks every function here against
golden vectors produced by the reference itself (tests/golden/make_golden.py,
run in the build container where /root/reference is importable).

The arithmetic follows the reference step by step so its CPU timing is a fair
stand-in for the reference: int32 numpy matmuls, a symmetric reduction after
every matrix product, channel chunks of accumulation_chunk(m), 64 positions
per GEMM batch and one worker thread per modulus.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from fractions import Fraction

import numpy as np

INT32_MAX = 2**31 - 1
POSITION_BATCH = 64   # rw/layer.py:248
INNER_BLOCK = 512     # rw/gemm.py:20


# ---------------------------------------------------------------------------
# residue helpers (rw/residue.py:27-47, rw/gemm.py:91-97, 25-33)

def sym(x: int, m: int) -> int:
    r = x % m
    return r - m if r > (m - 1) // 2 else r


def fold(a: np.ndarray, m: int) -> np.ndarray:
    """In-place symmetric reduction of an integer array."""
    np.mod(a, m, out=a)
    a[a > (m - 1) // 2] -= m
    return a


def narrow(m: int):
    return np.int8 if m < 256 else np.int16


def chunk_len(m: int) -> int:
    """Longest residue dot product that cannot overflow int32 (rw/gemm.py:30-33)."""
    h = (m - 1) // 2
    return (INT32_MAX - h) // (h * h)


# ---------------------------------------------------------------------------
# exact transforms (rw/transforms.py:58-256, 303-331), restated independently

def _points(n: int):
    pts = [Fraction(0)]
    k = 1
    while len(pts) < n - 1:
        pts += [Fraction(k), Fraction(-k)]
        k += 1
    return pts[: n - 1]  # finite points; infinity is implicit and last


def _poly_mul_linear(poly, root):
    out = [Fraction(0)] * (len(poly) + 1)
    for i, c in enumerate(poly):
        out[i + 1] += c
        out[i] -= root * c
    return out


def exact_matrices(m_out: int, r: int):
    """(AT, G, BT) as lists of Fractions for F(m_out, r) with default points."""
    n = m_out + r - 1
    fin = _points(n)
    # columns of the inverse Vandermonde: Lagrange bases, then prod(x - s)
    cols = []
    for j, s in enumerate(fin):
        poly, den = [Fraction(1)], Fraction(1)
        for k, t in enumerate(fin):
            if k != j:
                poly = _poly_mul_linear(poly, t)
                den *= s - t
        cols.append([c / den for c in poly] + [Fraction(0)])
    lead = [Fraction(1)]
    for t in fin:
        lead = _poly_mul_linear(lead, t)
    cols.append(lead)
    bt, g = [], []
    for k in range(n):
        lam = 1
        for v in cols[k]:
            lam = lam * v.denominator // math.gcd(lam, v.denominator)
        bt.append([v * lam for v in cols[k]])
        if k < n - 1:
            g.append([fin[k] ** e / lam for e in range(r)])
        else:
            g.append([Fraction(0)] * (r - 1) + [Fraction(1, lam)])
    at = [[fin[j] ** i for j in range(n - 1)] + [Fraction(1 if i == m_out - 1 else 0)] for i in range(m_out)]
    return at, g, bt


def modular_matrices(m_out: int, r: int, modulus: int):
    """(AT, G, BT) reduced mod ``modulus`` into symmetric narrow integers."""
    def red(rows):
        out = np.empty((len(rows), len(rows[0])), dtype=narrow(modulus))
        for i, row in enumerate(rows):
            for j, v in enumerate(row):
                out[i, j] = sym(v.numerator * pow(v.denominator, -1, modulus), modulus)
        return out
    return tuple(red(x) for x in exact_matrices(m_out, r))


# ---------------------------------------------------------------------------
# stage functions (rw/kernel.py:21-53, rw/layer.py:251-298)

def sandwich(left: np.ndarray, t: np.ndarray, right: np.ndarray, m: int) -> np.ndarray:
    a = fold(left.astype(np.int32) @ t.astype(np.int32), m)
    return fold(a @ right.astype(np.int32), m).astype(narrow(m))


def tile_conv_mod(g: np.ndarray, d: np.ndarray, m_out: int, r: int, modulus: int) -> np.ndarray:
    """rw/kernel.py:56-70: G g G^T, BT d BT^T, elementwise product, AT . AT^T,
    each reduced mod ``modulus`` (stacked tiles broadcast over leading dims)."""
    at, gm, bt = modular_matrices(m_out, r, modulus)
    u = sandwich(gm, g, gm.T, modulus).astype(np.int64)
    v = sandwich(bt, d, bt.T, modulus).astype(np.int64)
    return sandwich(at, fold(u * v, modulus), at.T, modulus)


def rns_tile_conv(g: np.ndarray, d: np.ndarray, m_out: int, r: int, moduli) -> np.ndarray:
    """rw/kernel.py:73-105: tile_conv_mod per modulus, then MRC."""
    outs = [tile_conv_mod(encode(g, q), encode(d, q), m_out, r, q) for q in moduli]
    return mrc(outs, moduli).astype(np.int32)


def encode(a: np.ndarray, m: int) -> np.ndarray:
    return fold(a.astype(np.int32), m).astype(narrow(m))


def patches_of(x: np.ndarray, m_out: int, r: int, pad: int):
    """Overlapping n x n patches at stride m_out on a zero canvas
    (rw/layer.py:118-158) -> (B, th, tw, n, n, C)."""
    b, h, w, c = x.shape
    n = m_out + r - 1
    oh, ow = h + 2 * pad - r + 1, w + 2 * pad - r + 1
    th, tw = -(-oh // m_out), -(-ow // m_out)
    canvas = np.zeros((b, (th - 1) * m_out + n, (tw - 1) * m_out + n, c), x.dtype)
    canvas[:, pad:pad + h, pad:pad + w] = x
    sb, sh, sw, sc = canvas.strides
    view = np.lib.stride_tricks.as_strided(
        canvas, shape=(b, th, tw, n, n, c), strides=(sb, sh * m_out, sw * m_out, sh, sw, sc), writeable=False)
    return np.ascontiguousarray(view), (oh, ow, th, tw)


def filter_bank(w: np.ndarray, mats: dict) -> dict:
    """{m: (n, n, C, K)} = G g G^T mod m (rw/layer.py:161-174)."""
    out = {}
    for m, (at, g, bt) in mats.items():
        u = sandwich(g, encode(w.transpose(2, 3, 0, 1), m), g.T, m)  # (C, K, n, n)
        out[m] = np.ascontiguousarray(u.transpose(2, 3, 0, 1))
    return out


def filter_bank_fast(w: np.ndarray, mats: dict) -> dict:
    """Same result as ``filter_bank`` (symmetric residues of G g G^T mod m),
    computed with two int64 einsums; used only to prepare CPU-baseline
    inputs quickly (the reference excludes the filter transform from its
    bench timing, rw/cli.py:459-463)."""
    out = {}
    r, _, c, k = w.shape
    wf = w.astype(np.float64).reshape(r, r * c * k)
    def fmod_sym(a, m):  # exact: integers < 2^52, x/m never ties for odd m
        a -= m * np.rint(a / m)
        return a

    for m, (at, g, bt) in mats.items():
        gf = g.astype(np.float64)  # products stay far below 2^53: exact
        t = fmod_sym((gf @ wf).reshape(-1, r, c * k), m)
        u = fmod_sym(np.matmul(gf[None], t), m)  # (n, n, c*k)
        out[m] = u.reshape(g.shape[0], g.shape[0], c, k).astype(narrow(m))
    return out


def input_stage(patches: np.ndarray, bt: np.ndarray, m: int) -> np.ndarray:
    """(B,th,tw,n,n,C) -> V (n*n, P, C)."""
    b, th, tw, n, _, c = patches.shape
    v = sandwich(bt, encode(patches.transpose(0, 1, 2, 5, 3, 4), m), bt.T, m)
    return np.ascontiguousarray(v.transpose(4, 5, 0, 1, 2, 3)).reshape(n * n, b * th * tw, c)


def residue_gemm(a: np.ndarray, b: np.ndarray, m: int) -> np.ndarray:
    """Stacked (a @ b) mod m, exact in int32 (rw/layer.py:251-263)."""
    acc = np.zeros(a.shape[:-1] + (b.shape[-1],), dtype=np.int32)
    step = chunk_len(m)
    for c0 in range(0, a.shape[-1], step):
        a_c, b_c = a[..., c0:c0 + step], b[..., c0:c0 + step, :]
        for k0 in range(0, a_c.shape[-1], INNER_BLOCK):
            acc += np.matmul(a_c[..., k0:k0 + INNER_BLOCK].astype(np.int32),
                             b_c[..., k0:k0 + INNER_BLOCK, :].astype(np.int32))
        fold(acc, m)
    return acc


def gemm_stage(vpos: np.ndarray, u: np.ndarray, m: int) -> np.ndarray:
    npos, p, c = vpos.shape
    k = u.shape[-1]
    upos = u.reshape(npos, c, k)
    acc = np.empty((npos, p, k), dtype=np.int32)
    for g0 in range(0, npos, POSITION_BATCH):
        acc[g0:g0 + POSITION_BATCH] = residue_gemm(vpos[g0:g0 + POSITION_BATCH], upos[g0:g0 + POSITION_BATCH], m)
    return acc


def output_stage(acc: np.ndarray, at: np.ndarray, m: int) -> np.ndarray:
    """(n*n, P, K) int32 -> y (P, K, m_out, m_out)."""
    npos, p, k = acc.shape
    n = int(round(npos ** 0.5))
    prod = np.ascontiguousarray(acc.reshape(n, n, p, k).transpose(2, 3, 0, 1)).astype(narrow(m))
    return sandwich(at, prod, at.T, m)


def mrc(residues, moduli) -> np.ndarray:
    """Mixed-radix reconstruction into the signed range (rw/residue.py:180-206)."""
    digits = []
    for j, m in enumerate(moduli):
        t = residues[j].astype(np.int64) % m
        for i in range(j):
            inv = sym(pow(moduli[i], -1, m), m)
            t = (t - digits[i]) * inv % m
        digits.append(t)
    x = digits[-1].copy()
    for j in range(len(moduli) - 2, -1, -1):
        x *= moduli[j]
        x += digits[j]
    d = math.prod(moduli)
    x[x > (d - 1) // 2] -= d
    return x


def winograd_layer(x: np.ndarray, w: np.ndarray, pad: int, m_out: int, moduli, mats: dict | None = None,
                   filters: dict | None = None, threads: int | None = None) -> np.ndarray:
    """The whole reference path: x (B,H,W,C) int8, w (R,R,C,K) int8 -> int32."""
    r, k = w.shape[0], w.shape[3]
    moduli = tuple(int(m) for m in moduli)
    if mats is None:
        mats = {m: modular_matrices(m_out, r, m) for m in moduli}
    patches, (oh, ow, th, tw) = patches_of(x, m_out, r, pad)
    if filters is None:
        filters = filter_bank(w, mats)

    def one(m):
        at, _, bt = mats[m]
        return output_stage(gemm_stage(input_stage(patches, bt, m), filters[m], m), at, m)

    workers = threads if threads is not None else int(os.environ.get("RNSW_THREADS", len(moduli)) or 1)
    workers = max(1, min(workers, len(moduli)))
    if workers > 1:
        with ThreadPoolExecutor(workers) as pool:
            ys = list(pool.map(one, moduli))
    else:
        ys = [one(m) for m in moduli]
    y = mrc(ys, moduli).astype(np.int32)
    b = x.shape[0]
    tiles = y.reshape(b, th, tw, k, m_out, m_out).transpose(0, 1, 4, 2, 5, 3)
    full = tiles.reshape(b, th * m_out, tw * m_out, k)
    return np.ascontiguousarray(full[:, :oh, :ow])


def direct_conv(x: np.ndarray, w: np.ndarray, pad: int) -> np.ndarray:
    """Exact int32 im2col convolution (rw/layer.py:81-103)."""
    b, h, wd, c = x.shape
    r, k = w.shape[0], w.shape[3]
    xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    win = np.lib.stride_tricks.sliding_window_view(xp, (r, r), axis=(1, 2))
    oh, ow = win.shape[1], win.shape[2]
    cols = np.ascontiguousarray(win.transpose(0, 1, 2, 4, 5, 3)).reshape(b * oh * ow, r * r * c)
    out = np.zeros((cols.shape[0], k), dtype=np.int32)
    wm = w.reshape(-1, k)
    for k0 in range(0, cols.shape[1], INNER_BLOCK):
        out += cols[:, k0:k0 + INNER_BLOCK].astype(np.int32) @ wm[k0:k0 + INNER_BLOCK].astype(np.int32)
    return out.reshape(b, oh, ow, k)
