"""Full-size BASELINE configs on the GPU, bit-exact against the reference:
output digests were computed by rnswinograd.winograd_layer_conv (and checked
equal to direct_conv) in tests/golden/make_golden.py."""
import numpy as np
import pytest

import oracle
from golden_util import digests, sha

pytestmark = pytest.mark.gpu


def _rnsw():
    import paper_2007_12216_b200 as rnsw

    return rnsw


def _run(case, w, x, layout="nhwc"):
    rnsw = _rnsw()
    spec = rnsw.LayerSpec(h=case.h, w=case.w, c=case.c, k=case.k, r=case.r, padding=case.pad, batch=case.batch,
                          tile_m=case.tile_m)
    return rnsw.winograd_layer_conv(spec, w, x, rnsw.RnsSystem(case.moduli), declared_bound=case.declared_bound)


def test_config1_bit_exact():
    from paper_2007_12216_b200 import workloads as W

    case, w, x = W.config1()
    y = _run(case, w, x)
    assert sha(y) == digests()["cfg1"]["y"]
    assert np.array_equal(y, oracle.direct_conv_c(x, w, case.pad))


def test_config1_nchw_front_door():
    from paper_2007_12216_b200 import workloads as W

    rnsw = _rnsw()
    case, w, x = W.config1()
    y = rnsw.conv2d_rns(np.ascontiguousarray(x.transpose(0, 3, 1, 2)), np.ascontiguousarray(w.transpose(3, 2, 0, 1)),
                        case.moduli, case.tile_m, case.pad, declared_bound=case.declared_bound)
    assert sha(np.ascontiguousarray(y.transpose(0, 2, 3, 1))) == digests()["cfg1"]["y"]


def test_config3_bit_exact():
    from paper_2007_12216_b200 import workloads as W

    case, w, x = W.config3()
    y = _run(case, w, x)
    assert sha(y) == digests()["cfg3"]["y"]
    assert np.array_equal(y, oracle.direct_conv_c(x, w, case.pad))


@pytest.mark.parametrize("idx", range(13))
def test_config5_sweep_bit_exact(idx):
    from paper_2007_12216_b200 import workloads as W

    case = W.config5_cases()[idx]
    w, x = W.config5_operands()
    y = _run(case, w, x)
    d = digests()
    assert sha(y) == d[case.name]["y"] == d["cfg5/direct"]["y"], case.name


def test_vgg16_batch1_every_layer_bit_exact():
    """Config 2: all 13 layers' int32 outputs and the final map match the
    reference RNS path (and direct conv) byte for byte."""
    import torch
    from paper_2007_12216_b200 import workloads as W
    from paper_2007_12216_b200.vgg import VGG16Rns

    net = VGG16Rns()
    x = torch.from_numpy(W.vgg16_images(1)).cuda()
    final, outs = net.forward(x, keep_int32=True)
    d = digests()
    for (name, *_), y in zip(W.VGG16_LAYERS, outs):
        assert sha(y.cpu().numpy()) == d[f"vgg16/{name}"]["y"], name
    assert sha(final.cpu().numpy()) == d["vgg16/final"]["y"]


def test_vgg16_batch4_matches_per_image_runs():
    import torch
    from paper_2007_12216_b200 import workloads as W
    from paper_2007_12216_b200.vgg import VGG16Rns

    net = VGG16Rns()
    xb = torch.from_numpy(W.vgg16_images(4)).cuda()
    full = net.forward(xb).cpu().numpy()
    for i in range(4):
        one = net.forward(torch.from_numpy(W.vgg16_images(1, start=i)).cuda()).cpu().numpy()
        assert np.array_equal(full[i:i + 1], one)
    staged = net.forward_staged(xb, lambda *a: None).cpu().numpy()
    assert np.array_equal(staged, full)


def test_vgg16_fused_glue_matches_unfused():
    """The fused requant/pool epilogue (rnsw_conv_forward_requant) gives the
    same int8 maps as int32 output + separate glue, layer by layer."""
    import torch
    from paper_2007_12216_b200 import workloads as W
    from paper_2007_12216_b200.vgg import VGG16Rns

    net = VGG16Rns()
    x = torch.from_numpy(W.vgg16_images(3)).cuda()
    a = net.forward(x).cpu().numpy()
    b = net.forward_fused(x).cpu().numpy()
    c = net.forward_fused_staged(x, lambda *args: None).cpu().numpy()
    assert np.array_equal(a, b) and np.array_equal(a, c)
    one = net.forward_fused(x[:1]).cpu().numpy()
    assert sha(one) == digests()["vgg16/final"]["y"]


def test_vgg16_batch256_matches_single_image_runs():
    """The bench workload itself (config 4, B=256, fused, CUDA graph): sampled
    images equal their own batch-1 runs, which are pinned to the reference
    digests -- no cross-tile / cross-image interference at full scale."""
    import torch
    from paper_2007_12216_b200 import workloads as W
    from paper_2007_12216_b200.vgg import VGG16Rns

    net = VGG16Rns()
    x = torch.from_numpy(W.vgg16_images(256)).cuda()
    out = net.graph(x)(x).cpu()
    for i in (0, 1, 127, 128, 255):
        one = net.forward_fused(x[i:i + 1].contiguous()).cpu()
        assert torch.equal(out[i:i + 1], one), i
    assert sha(out[:1].numpy()) == digests()["vgg16/final"]["y"]


def test_vgg16_streamed_serving_matches_forward():
    """VGG16Rns.run_stream (copies overlapped with compute, CUDA graphs bound
    to two input buffers) returns the same maps as forward_fused per batch."""
    import torch
    from paper_2007_12216_b200 import workloads as W
    from paper_2007_12216_b200.vgg import VGG16Rns

    net = VGG16Rns()
    batches = [torch.from_numpy(W.vgg16_images(2, start=2 * i)).pin_memory() for i in range(4)]
    outs = [torch.empty((2, 7, 7, 512), dtype=torch.int8).pin_memory() for _ in range(4)]
    net.run_stream(batches, outs)
    torch.cuda.synchronize()
    for b, o in zip(batches, outs):
        assert torch.equal(o, net.forward_fused(b.cuda()).cpu())
    assert sha(outs[0][:1].numpy()) == digests()["vgg16/final"]["y"]


def test_fused_requant_single_layers():
    import torch
    from oracle.vgg_ref import requant_pool
    from paper_2007_12216_b200 import _native
    from paper_2007_12216_b200.layer import _filters_on_device, _stream_ptr, plan_for
    import paper_2007_12216_b200 as rnsw

    rng = np.random.default_rng(77)
    for (h, c, k, tm, pool, shift) in [(28, 32, 64, 14, 1, 9), (20, 16, 36, 6, 0, 7), (17, 48, 8, 8, 1, 11),
                                       (12, 64, 20, 10, 1, 8)]:
        system = rnsw.RnsSystem((4001, 4331) if tm % 2 == 0 and tm > 8 else (251, 241, 239))
        plan = plan_for(rnsw.cached_transforms(tm, 3), system)
        x = rng.integers(0, 128, (2, h, h, c)).astype(np.int8)
        w = np.clip(np.rint(rng.normal(0, 20, (3, 3, c, k))), -127, 127).astype(np.int8)
        bank = _filters_on_device(plan, torch.from_numpy(w).cuda(), c, k, _native.LAYOUT_NHWC)
        l = _native.lib()
        ws_bytes = l.rnsw_workspace_bytes(plan.handle, 2, h, h, c, k, 1)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
        oh = h // 2 if pool else h
        out = torch.empty((2, oh, oh, k), dtype=torch.int8, device="cuda")
        xd = torch.from_numpy(x).cuda()
        vp = _native.c_void_p
        _native.check(l.rnsw_conv_forward_requant(plan.handle, vp(xd.data_ptr()), 2, h, h, c, k, 1,
                                                  vp(bank.data.data_ptr()), shift, pool, vp(out.data_ptr()),
                                                  vp(ws.data_ptr()), ws_bytes, _stream_ptr()))
        want = requant_pool(oracle.direct_conv_c(x, w, 1), shift, bool(pool))
        assert np.array_equal(out.cpu().numpy(), want), (h, c, k, tm, pool)


@pytest.mark.skipif(__import__("os").environ.get("RNSW_K4_NO_Z3") is not None, reason="already the alternate path")
def test_alternate_kernel_paths_in_subprocess():
    """The A/B switches read once per process (RNSW_K4_MMA_SYNC: the mma.sync
    output transform instead of the tcgen05 one; RNSW_K4_NO_Z3: it with a
    reduced pass 1 instead of the three-limb pass 2; RNSW_GEMM_NO_MC: GEMM
    without CTA pairs) select kernels the default dispatch does not use for
    the VGG16 shapes: rerun the VGG16 and fused-epilogue checks on them."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, RNSW_K4_NO_Z3="1", RNSW_GEMM_NO_MC="1", RNSW_K4_MMA_SYNC="1")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_configs.py"),
                        "-k", "vgg16_batch1 or fused_glue or fused_requant or config5_sweep"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.skipif(__import__("os").environ.get("RNSW_GEMM_CG2") is not None, reason="already forced")
@pytest.mark.parametrize("cg2", ["0", "1"])
def test_gemm_pair_modes_in_subprocess(cg2):
    """RNSW_GEMM_CG2=1 runs every paired 16-bit GEMM as cta_group::2 MMAs of
    M = 256 (default only for C >= 256), =0 every pair as a multicast pair:
    rerun the VGG16 batch checks and the fused-epilogue sweep on each."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, RNSW_GEMM_CG2=cg2)
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_configs.py"),
                        "-k", "vgg16_batch or fused_glue or fused_requant"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.skipif(__import__("os").environ.get("RNSW_K4_STG_STORES") is not None, reason="already forced")
def test_k4_per_thread_stores_in_subprocess():
    """RNSW_K4_STG_STORES=1 keeps the two-pass output transform's per-thread
    16-byte stores instead of its TMA bulk tensor store of each staged tile:
    rerun the fused-glue checks (pooled and unpooled int8 tiles, ragged
    edges) on that path."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, RNSW_K4_STG_STORES="1")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_configs.py"), "-k", "vgg16_batch1 or fused_glue or fused_requant"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
