"""Per-stage device entry points with reference-layout views.

Each function runs ONE device stage through the C ABI and returns its result
in the layout of the matching reference function, so every stage can be
checked on its own:

    input_transform   ~ _modulus_pass part 1   -> {m: vpos (N*N, P, C)}   (rw/layer.py:278-283)
    winograd_gemm     ~ _modular_gemm loop     -> {m: acc  (N*N, P, K)}   (rw/layer.py:285-291)
    output_residues   ~ backward_transform_mod -> {m: y    (P, K, M, M)}  (rw/layer.py:293-297)
    mrc_reconstruct   ~ mrc_reconstruct_arrays -> int64                   (rw/residue.py:180-206)

The views only reinterpret device buffers (limb planes -> int16); all
arithmetic is done by the kernels.
"""

from __future__ import annotations

from math import ceil

from . import _native
from .layer import _stream_ptr, plan_for, to_device
from .transforms import cached_transforms


def _torch():
    import torch

    return torch


def _plan(tile_m, r, system):
    return plan_for(cached_transforms(tile_m, r), system)


def _cp(c: int) -> int:
    return 32 if c <= 32 else 64 if c <= 64 else (c + 127) // 128 * 128


def planes_to_residues(buf, plan, rows: int, cols: int, cols_padded: int) -> dict:
    """[plane][pos][rows][cols_padded] int8 limb planes -> {m: (pos, rows, cols) int16}."""
    torch = _torch()
    n2 = plan.n * plan.n
    v = buf.view(torch.int8)[: plan.n_planes * n2 * rows * cols_padded]
    v = v.view(plan.n_planes, n2, rows, cols_padded)[..., :cols]
    out, base = {}, 0
    for m in plan.moduli:
        val = v[base].to(torch.int16)
        if m >= 256:
            val = v[base + 1].to(torch.int16) * 256 + val
            base += 2
        else:
            base += 1
        out[m] = val
    return out


def input_transform(x, tile_m: int, r: int, system, padding: int, layout: int = _native.LAYOUT_NHWC):
    """Returns (raw V buffer, {m: vpos (N*N, P, C) int16}, P)."""
    torch = _torch()
    l = _native.lib()
    plan = _plan(tile_m, r, system)
    xd = to_device(x)
    if layout == _native.LAYOUT_NHWC:
        b, h, w, c = xd.shape
    else:
        b, c, h, w = xd.shape
    ho, wo = h + 2 * padding - r + 1, w + 2 * padding - r + 1
    p = b * ceil(ho / tile_m) * ceil(wo / tile_m)
    nbytes = l.rnsw_v_bytes(plan.handle, p, c)
    buf = torch.empty(nbytes, dtype=torch.uint8, device=xd.device)
    _native.check(l.rnsw_input_transform(plan.handle, _native.c_void_p(xd.data_ptr()), b, h, w, c, padding, layout,
                                         _native.c_void_p(buf.data_ptr()), nbytes, _stream_ptr()))
    return buf, planes_to_residues(buf, plan, p, c, _cp(c)), p


def winograd_gemm(vbuf, bank, tile_m: int, r: int, system, p: int, c: int, k: int):
    """Returns (raw Mw buffer, {m: acc (N*N, P, K) int16})."""
    torch = _torch()
    l = _native.lib()
    plan = _plan(tile_m, r, system)
    nbytes = l.rnsw_m_bytes(plan.handle, p, k)
    mw = torch.empty(nbytes, dtype=torch.uint8, device=vbuf.device)
    _native.check(l.rnsw_winograd_gemm(plan.handle, _native.c_void_p(vbuf.data_ptr()),
                                       _native.c_void_p(bank.data_ptr()), p, c, k, _native.c_void_p(mw.data_ptr()),
                                       nbytes, _stream_ptr()))
    kp = (k + 15) // 16 * 16
    n2 = plan.n * plan.n
    # blocked layout [ceil(P/128)][res][pos][128][Kp] (include/rnsw.h)
    nb = (p + 127) // 128
    view = mw.view(torch.int16)[: nb * len(plan.moduli) * n2 * 128 * kp].view(nb, len(plan.moduli), n2, 128, kp)
    view = view.permute(1, 2, 0, 3, 4).reshape(len(plan.moduli), n2, nb * 128, kp)[:, :, :p, :k]
    return mw, {m: view[i] for i, m in enumerate(plan.moduli)}


def output_residues(mw, tile_m: int, r: int, system, p: int, k: int):
    """{m: (P, K, M, M) int16} residues of AT M A mod m."""
    torch = _torch()
    l = _native.lib()
    plan = _plan(tile_m, r, system)
    out = torch.empty((len(plan.moduli), p, k, tile_m, tile_m), dtype=torch.int16, device=mw.device)
    _native.check(l.rnsw_output_residues(plan.handle, _native.c_void_p(mw.data_ptr()), p, k,
                                         _native.c_void_p(out.data_ptr()), _stream_ptr()))
    return {m: out[i] for i, m in enumerate(plan.moduli)}


def mrc_reconstruct(residues, tile_m: int, r: int, system):
    """residues: (n_res, count) int16 device tensor -> int64 (count,)."""
    torch = _torch()
    l = _native.lib()
    plan = _plan(tile_m, r, system)
    res = to_device(residues).to(torch.int16).contiguous()
    out = torch.empty(res.shape[1], dtype=torch.int64, device=res.device)
    _native.check(l.rnsw_mrc_reconstruct(plan.handle, _native.c_void_p(res.data_ptr()), res.shape[1],
                                         _native.c_void_p(out.data_ptr()), _stream_ptr()))
    return out
