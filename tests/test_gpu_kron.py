"""The Kronecker output transform on tcgen05 (csrc/output_kron.cu: one
GEMM per residue and row block, A = kron(AT, AT) resident in TMEM, residue
exchange through distributed shared memory for the mixed-radix
reconstruction) against the exact direct convolution and the oracle, on every
16-bit tile it serves and in all three output modes (int32, requantised int8,
requantised + 2x2 max-pooled int8)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from oracle import ref_port as O

pytestmark = pytest.mark.gpu

SYS16 = (4001, 4331)


@pytest.mark.parametrize("tile_m", [2, 4, 6, 8, 10, 12, 14])
@pytest.mark.parametrize("h,w,c,k,b", [(30, 23, 32, 64, 2), (17, 17, 64, 48, 1), (9, 40, 16, 16, 3)])
def test_int32_layer(tile_m, h, w, c, k, b):
    import paper_2007_12216_b200 as rnsw

    rng = np.random.default_rng(tile_m * 100 + h + k)
    wt = rng.integers(-128, 128, (3, 3, c, k)).astype(np.int8)
    x = rng.integers(-128, 128, (b, h, w, c)).astype(np.int8)
    spec = rnsw.LayerSpec(h=h, w=w, c=c, k=k, r=3, padding=1, batch=b, tile_m=tile_m)
    system = rnsw.RnsSystem(SYS16)
    got = rnsw.winograd_layer_conv(spec, wt, x, system, declared_bound=system.signed_bound)
    assert np.array_equal(got, O.winograd_layer(x, wt, 1, tile_m, SYS16))
    assert np.array_equal(got, oracle.direct_conv_c(x, wt, 1))


@pytest.mark.parametrize("tile_m,pool,shift", [(14, 1, 9), (14, 0, 8), (12, 1, 10), (10, 0, 9), (8, 1, 9), (6, 1, 8)])
@pytest.mark.parametrize("h,c,k", [(28, 32, 64), (31, 64, 128), (15, 16, 32)])
def test_requant_layer(tile_m, pool, shift, h, c, k):
    import torch
    from oracle.vgg_ref import requant_pool
    from paper_2007_12216_b200 import _native
    from paper_2007_12216_b200.layer import _filters_on_device, _stream_ptr, plan_for
    import paper_2007_12216_b200 as rnsw

    rng = np.random.default_rng(tile_m + h + c)
    b = 2
    plan = plan_for(rnsw.cached_transforms(tile_m, 3), rnsw.RnsSystem(SYS16))
    x = rng.integers(0, 128, (b, h, h, c)).astype(np.int8)
    w = np.clip(np.rint(rng.normal(0, 20, (3, 3, c, k))), -127, 127).astype(np.int8)
    bank = _filters_on_device(plan, torch.from_numpy(w).cuda(), c, k, _native.LAYOUT_NHWC)
    l = _native.lib()
    ws_bytes = l.rnsw_workspace_bytes(plan.handle, b, h, h, c, k, 1)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    oh = h // 2 if pool else h
    out = torch.full((b, oh, oh, k), 77, dtype=torch.int8, device="cuda")
    xd = torch.from_numpy(x).cuda()
    vp = _native.c_void_p
    _native.check(l.rnsw_conv_forward_requant(plan.handle, vp(xd.data_ptr()), b, h, h, c, k, 1,
                                              vp(bank.data.data_ptr()), shift, pool, vp(out.data_ptr()),
                                              vp(ws.data_ptr()), ws_bytes, _stream_ptr()))
    want = requant_pool(oracle.direct_conv_c(x, w, 1), shift, bool(pool))
    assert np.array_equal(out.cpu().numpy(), want)


def test_wrap_beyond_dynamic_range():
    """A false declared bound wraps modulo D exactly like the reference."""
    import paper_2007_12216_b200 as rnsw

    spec = rnsw.LayerSpec(h=16, w=16, c=512, k=16, r=3, padding=1, batch=1, tile_m=14)
    rng = np.random.default_rng(4)
    w = np.where(rng.random(spec.weight_shape()) < 0.5, -128, 127).astype(np.int8)
    x = np.where(rng.random(spec.input_shape()) < 0.5, -128, 127).astype(np.int8)
    system = rnsw.RnsSystem(SYS16)
    y = rnsw.winograd_layer_conv(spec, w, x, system, declared_bound=system.signed_bound)
    d = oracle.direct_conv_c(x, w, 1).astype(np.int64)
    D = 4001 * 4331
    assert np.array_equal(y.astype(np.int64), ((d + D // 2) % D) - D // 2)


@pytest.mark.skipif(os.environ.get("RNSW_K4_TWO_PASS") is not None, reason="already the alternate path")
def test_two_pass_output_transform_still_matches():
    """RNSW_K4_TWO_PASS=1 keeps the two-pass kernels (output_umma.cu /
    output_tc.cu): rerun this file's checks on them in a subprocess."""
    env = dict(os.environ, RNSW_K4_TWO_PASS="1")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_kron.py"), "-k", "int32_layer or requant_layer"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


SYS8 = (251, 241, 239)


@pytest.mark.parametrize("mods", [SYS8, (253, 251, 247), (251, 241), (251,), (7, 11, 13), (7, 11, 13, 17)])
@pytest.mark.parametrize("tile_m,r", [(6, 3), (8, 3), (10, 3), (12, 3), (14, 3), (8, 5), (4, 3)])
def test_int32_layer_8bit(mods, tile_m, r):
    """8-bit residue systems (1-4 residues): every residue of a row block in
    one CTA, mixed-radix digits folded into the reductions."""
    import paper_2007_12216_b200 as rnsw

    system = rnsw.RnsSystem(mods)
    try:
        rnsw.reduce_for_system(rnsw.cached_transforms(tile_m, r), system)
    except rnsw.NotCoprime:
        pytest.skip(f"moduli {mods} not compatible with F({tile_m},{r})")
    rng = np.random.default_rng(tile_m * 7 + len(mods))
    b, h, w, c, k = 2, 21, 17, 32, 48
    wt = rng.integers(-128, 128, (r, r, c, k)).astype(np.int8)
    x = rng.integers(-128, 128, (b, h, w, c)).astype(np.int8)
    pad = r // 2
    spec = rnsw.LayerSpec(h=h, w=w, c=c, k=k, r=r, padding=pad, batch=b, tile_m=tile_m)
    got = rnsw.winograd_layer_conv(spec, wt, x, system, declared_bound=system.signed_bound)
    assert np.array_equal(got, O.winograd_layer(x, wt, pad, tile_m, mods))


@pytest.mark.parametrize("tile_m,pool", [(8, 1), (10, 0), (6, 1), (14, 1)])
def test_requant_layer_8bit(tile_m, pool):
    import torch
    from oracle.vgg_ref import requant_pool
    from paper_2007_12216_b200 import _native
    from paper_2007_12216_b200.layer import _filters_on_device, _stream_ptr, plan_for
    import paper_2007_12216_b200 as rnsw

    rng = np.random.default_rng(tile_m)
    b, h, c, k, shift = 2, 30, 64, 32, 8
    plan = plan_for(rnsw.cached_transforms(tile_m, 3), rnsw.RnsSystem(SYS8))
    x = rng.integers(0, 128, (b, h, h, c)).astype(np.int8)
    w = rng.integers(-8, 9, (3, 3, c, k)).astype(np.int8)
    bank = _filters_on_device(plan, torch.from_numpy(w).cuda(), c, k, _native.LAYOUT_NHWC)
    l = _native.lib()
    ws_bytes = l.rnsw_workspace_bytes(plan.handle, b, h, h, c, k, 1)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    oh = h // 2 if pool else h
    out = torch.full((b, oh, oh, k), 77, dtype=torch.int8, device="cuda")
    xd = torch.from_numpy(x).cuda()
    vp = _native.c_void_p
    _native.check(l.rnsw_conv_forward_requant(plan.handle, vp(xd.data_ptr()), b, h, h, c, k, 1,
                                              vp(bank.data.data_ptr()), shift, pool, vp(out.data_ptr()),
                                              vp(ws.data_ptr()), ws_bytes, _stream_ptr()))
    want = requant_pool(oracle.direct_conv_c(x, w, 1), shift, bool(pool))
    assert np.array_equal(out.cpu().numpy(), want)
