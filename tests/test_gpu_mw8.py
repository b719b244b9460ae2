"""The Mw8 path (F(14x14,3x3) over RNS(4001,4331)): the tcgen05 output
transform fed synthetic Winograd-domain products checked against numpy, and
the _mw8 stage calls chained equal to the whole-layer call and the oracle."""
import numpy as np
import pytest

import oracle
from oracle.vgg_ref import requant_pool

pytestmark = pytest.mark.gpu

MODS = (4001, 4331)


def _setup():
    import paper_2007_12216_b200 as rnsw
    from paper_2007_12216_b200.layer import plan_for

    ts = rnsw.cached_transforms(14, 3)
    system = rnsw.RnsSystem(MODS)
    return rnsw, ts, system, plan_for(ts, system)


def _expected(rnsw, ts, system, mat, B, H, W, K):
    """numpy restatement of Y = AT M AT^T mod m, mixed radix, crop
    (rw/kernel.py:50-53, rw/residue.py:180-206, rw/layer.py:378-388)."""
    mts = rnsw.transforms.reduce_for_system(ts, system)
    P = mat.shape[1]
    yr = []
    for r, m in enumerate(MODS):
        at = mts[r].at.astype(np.int64)
        yr.append(np.einsum("ai,pijk,bj->pabk", at, mat[r].reshape(P, 16, 16, K), at) % m)
    m0, m1 = MODS
    d1 = ((yr[1] - yr[0]) * pow(m0, -1, m1)) % m1
    x = yr[0] + m0 * d1
    x = np.where(x > (m0 * m1 - 1) // 2, x - m0 * m1, x)
    th, tw = -(-H // 14), -(-W // 14)
    out = np.zeros((B, th * 14, tw * 14, K), np.int64)
    for p in range(P):
        b, rem = divmod(p, th * tw)
        ti, tj = divmod(rem, tw)
        out[b, ti * 14:ti * 14 + 14, tj * 14:tj * 14 + 14] = x[p]
    return out[:, :H, :W].astype(np.int32)


def _mw8_bytes(mat, Kp):
    P = mat.shape[1]
    K = mat.shape[3]
    num_pb = -(-P // 128)
    buf = np.zeros((num_pb, 2, 2, 256, 128, Kp), np.uint8)
    for p in range(P):
        for r in range(2):
            buf[p >> 7, r, 0, :, p & 127, :K] = mat[r, p] & 255
            buf[p >> 7, r, 1, :, p & 127, :K] = mat[r, p] >> 8
    return buf.reshape(-1)


@pytest.mark.parametrize("B,H,W,K,layout", [(1, 28, 28, 32, 0), (2, 17, 30, 40, 0), (1, 14, 15, 7, 1),
                                             (3, 9, 9, 64, 1), (1, 150, 20, 16, 0)])
def test_output_transform_mw8_against_numpy(B, H, W, K, layout):
    import torch
    from paper_2007_12216_b200 import _native
    from paper_2007_12216_b200.layer import _stream_ptr

    rnsw, ts, system, plan = _setup()
    l = _native.lib()
    assert l.rnsw_mw8_supported(plan.handle) == 1
    P = B * (-(-H // 14)) * (-(-W // 14))
    Kp = -(-K // 16) * 16
    rng = np.random.default_rng(B * 1000 + H * 10 + K)
    mat = np.stack([rng.integers(0, m, (P, 256, K)) for m in MODS])
    mat[:, 0, :3] = np.array([m - 1 for m in MODS])[:, None, None]  # extremes
    dev = torch.from_numpy(_mw8_bytes(mat, Kp)).cuda()
    shape = (B, H, W, K) if layout == 0 else (B, K, H, W)
    y = torch.zeros(shape, dtype=torch.int32, device="cuda")
    _native.check(l.rnsw_output_transform_mw8(plan.handle, _native.c_void_p(dev.data_ptr()), B, H, W, K, 1, layout,
                                              _native.c_void_p(y.data_ptr()), _stream_ptr()))
    got = y.cpu().numpy()
    if layout == 1:
        got = got.transpose(0, 2, 3, 1)
    assert np.array_equal(got, _expected(rnsw, ts, system, mat, B, H, W, K))


@pytest.mark.parametrize("c,k,h,pool,shift", [(3, 64, 30, 1, 9), (32, 48, 28, 0, 8), (64, 96, 20, 1, 10),
                                             (16, 20, 30, 0, 7), (16, 36, 18, 1, 8)])
def test_mw8_stage_chain_equals_layer_and_oracle(c, k, h, pool, shift):
    import torch
    from paper_2007_12216_b200 import _native
    from paper_2007_12216_b200.layer import _filters_on_device, _stream_ptr

    rnsw, ts, system, plan = _setup()
    l = _native.lib()
    vp = _native.c_void_p
    rng = np.random.default_rng(c + k + h)
    x = rng.integers(0, 128, (2, h, h, c)).astype(np.int8)
    w = np.clip(np.rint(rng.normal(0, 20, (3, 3, c, k))), -127, 127).astype(np.int8)
    bank = _filters_on_device(plan, torch.from_numpy(w).cuda(), c, k, _native.LAYOUT_NHWC)
    xd = torch.from_numpy(x).cuda()
    s = _stream_ptr()
    ws_bytes = l.rnsw_workspace_bytes(plan.handle, 2, h, h, c, k, 1)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    tiles = 2 * (-(-h // 14)) ** 2
    vb = (l.rnsw_v_bytes(plan.handle, tiles, c) + 255) // 256 * 256
    v_ptr, m_ptr, mb = ws.data_ptr(), ws.data_ptr() + vb, ws_bytes - vb
    if c <= 4:
        _native.check(l.rnsw_input_transform_compact(plan.handle, vp(xd.data_ptr()), 2, h, h, c, 1, 0, vp(v_ptr),
                                                     vb, s))
        _native.check(l.rnsw_small_channel_product_mw8(plan.handle, vp(v_ptr), vp(bank.data.data_ptr()), tiles, c,
                                                       k, vp(m_ptr), mb, s))
    else:
        _native.check(l.rnsw_input_transform(plan.handle, vp(xd.data_ptr()), 2, h, h, c, 1, 0, vp(v_ptr), vb, s))
        _native.check(l.rnsw_winograd_gemm_mw8(plan.handle, vp(v_ptr), vp(bank.data.data_ptr()), tiles, c, k,
                                               vp(m_ptr), mb, s))
    y = torch.empty((2, h, h, k), dtype=torch.int32, device="cuda")
    _native.check(l.rnsw_output_transform_mw8(plan.handle, vp(m_ptr), 2, h, h, k, 1, 0, vp(y.data_ptr()), s))
    oh = h // 2 if pool else h
    q = torch.empty((2, oh, oh, k), dtype=torch.int8, device="cuda")
    _native.check(l.rnsw_output_transform_requant_mw8(plan.handle, vp(m_ptr), 2, h, h, k, 1, shift, pool,
                                                      vp(q.data_ptr()), s))
    want = oracle.direct_conv_c(x, w, 1)
    assert np.array_equal(y.cpu().numpy(), want)
    assert np.array_equal(q.cpu().numpy(), requant_pool(want, shift, bool(pool)))
    y2 = torch.empty_like(y)
    _native.check(l.rnsw_conv_forward(plan.handle, vp(xd.data_ptr()), 2, h, h, c, k, 1, 0, vp(bank.data.data_ptr()),
                                      vp(y2.data_ptr()), vp(ws.data_ptr()), ws_bytes, s))
    assert torch.equal(y, y2)


def test_mw8_unsupported_plans_refuse():
    import paper_2007_12216_b200 as rnsw
    from paper_2007_12216_b200 import _native
    from paper_2007_12216_b200.layer import plan_for

    l = _native.lib()
    plan8 = plan_for(rnsw.cached_transforms(8, 3), rnsw.RnsSystem((251, 241, 239)))
    assert l.rnsw_mw8_supported(plan8.handle) == 0
    rc = l.rnsw_output_transform_mw8(plan8.handle, _native.c_void_p(16), 1, 8, 8, 16, 1, 0, _native.c_void_p(16),
                                     None)
    assert rc != 0 and b"Mw8" in l.rnsw_last_error()


def test_mw8_moduli_near_the_fast_limit():
    """RNS(4493, 4489) at F(14,3): the largest 16-bit moduli the tcgen05 output
    transform takes (m < 4500), where its bias and limb bounds are tightest;
    extreme and random int8 operands against direct conv and the oracle."""
    import paper_2007_12216_b200 as rnsw
    from oracle import ref_port
    from paper_2007_12216_b200 import _native
    from paper_2007_12216_b200.layer import plan_for

    system = rnsw.RnsSystem((4493, 4489))
    plan = plan_for(rnsw.cached_transforms(14, 3), system)
    assert _native.lib().rnsw_mw8_supported(plan.handle) == 1
    spec = rnsw.LayerSpec(h=30, w=30, c=64, k=32, r=3, padding=1, tile_m=14)
    rng = np.random.default_rng(4493)
    cases = [(rng.integers(-128, 128, spec.input_shape()), rng.integers(-127, 128, spec.weight_shape())),
             (np.full(spec.input_shape(), -128), np.full(spec.weight_shape(), 127)),
             (np.full(spec.input_shape(), 127), np.where(rng.random(spec.weight_shape()) < 0.5, -127, 127))]
    for x, w in cases:
        x, w = x.astype(np.int8), w.astype(np.int8)
        got = rnsw.winograd_layer_conv(spec, w, x, system)
        assert np.array_equal(got, oracle.direct_conv_c(x, w, 1))
    assert np.array_equal(got, ref_port.winograd_layer(x, w, 1, 14, system.moduli))
