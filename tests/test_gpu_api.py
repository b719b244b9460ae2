"""The reference-facing API on the GPU: operand types, precomputed filters,
timings, declared-bound wrap semantics, edge geometries and worst-case values.
Every result is compared with the CPU oracle (reference restatement) and the
exact direct convolution."""
import numpy as np
import pytest

import oracle
from oracle import ref_port as O

pytestmark = pytest.mark.gpu


def _rnsw():
    import paper_2007_12216_b200 as rnsw

    return rnsw


def _operands(spec, seed, lo=-128, hi=127):
    rng = np.random.default_rng(seed)
    return (rng.integers(lo, hi + 1, spec.weight_shape()).astype(np.int8),
            rng.integers(lo, hi + 1, spec.input_shape()).astype(np.int8))


EDGE = [
    # h, w, c, k, r, pad, batch, tile_m, moduli
    (3, 3, 1, 1, 3, 0, 1, 4, (251, 241, 239)),          # single output pixel, tile larger than output
    (5, 17, 2, 1, 3, 1, 3, 6, (4001, 4331)),            # ragged width, K = 1
    (7, 7, 17, 33, 5, 2, 2, 12, (4001, 4331)),          # N = 16 with R = 5, odd C and K
    (33, 31, 64, 48, 3, 1, 5, 8, (253, 251, 247)),      # P not a multiple of 128
    (14, 14, 512, 16, 3, 1, 1, 14, (4001, 4331)),       # deep C (4 chunks of 128)
    (9, 9, 130, 300, 3, 1, 1, 10, (251, 241, 239)),     # C -> Cp = 256, K padded to 304
    (10, 12, 40, 24, 3, 2, 2, 6, (251, 241, 239)),      # padding 2 with R = 3
    (6, 6, 8, 8, 3, 0, 200, 4, (7, 11, 13)),            # many tiny tiles, tiny moduli
    (20, 20, 16, 16, 3, 1, 1, 2, (251, 241, 239, 233)), # four residues, F(2,3)
]


@pytest.mark.parametrize("case", EDGE, ids=lambda c: "x".join(map(str, c[:8])))
def test_edge_geometries(case):
    rnsw = _rnsw()
    h, w, c, k, r, pad, batch, tm, mods = case
    spec = rnsw.LayerSpec(h=h, w=w, c=c, k=k, r=r, padding=pad, batch=batch, tile_m=tm)
    system = rnsw.RnsSystem(mods)
    lo, hi = (-2, 2) if max(mods) < 20 else (-128, 127)
    wt, x = _operands(spec, h * 7 + c, lo, hi)
    got = rnsw.winograd_layer_conv(spec, wt, x, system, declared_bound=system.signed_bound)
    assert np.array_equal(got, O.winograd_layer(x, wt, pad, tm, mods))
    direct = oracle.direct_conv_c(x, wt, pad)
    if np.abs(direct.astype(np.int64)).max() <= system.signed_bound:
        assert np.array_equal(got, direct)


def test_worst_case_extremes():
    """All operands at the int8 extremes -128 / 127 (t/test_kernel.py:191-199)."""
    rnsw = _rnsw()
    spec = rnsw.LayerSpec(h=12, w=12, c=8, k=4, r=3, padding=1, tile_m=10)
    for xv, wv in [(-128, 127), (-128, -128), (127, 127)]:
        x = np.full(spec.input_shape(), xv, np.int8)
        w = np.full(spec.weight_shape(), wv, np.int8)
        system = rnsw.RnsSystem((4001, 4331))
        got = rnsw.winograd_layer_conv(spec, w, x, system, declared_bound=9 * 8 * 128 * 128)
        assert np.array_equal(got, oracle.direct_conv_c(x, w, 1))


def test_declared_bound_wraps_like_the_reference():
    """A false declared bound wraps modulo D exactly as the reference does
    (SURVEY.md finding 3): same output as the reference path, congruent to
    direct conv, not equal to it."""
    rnsw = _rnsw()
    spec = rnsw.LayerSpec(h=8, w=8, c=64, k=8, r=3, padding=1, tile_m=4)
    w, x = _operands(spec, 3)
    system = rnsw.RnsSystem((7, 11, 13))
    got = rnsw.winograd_layer_conv(spec, w, x, system, declared_bound=100)
    assert np.array_equal(got, O.winograd_layer(x, w, 1, 4, (7, 11, 13)))
    direct = oracle.direct_conv_c(x, w, 1).astype(np.int64)
    assert np.all((direct - got) % 1001 == 0) and not np.array_equal(got, direct)


def test_declared_bound_at_512_channels():
    # t/test_layer.py:181-194: ternary weights keep |y| < 300000 at C = 512
    rnsw = _rnsw()
    spec = rnsw.LayerSpec(h=6, w=6, c=512, k=4, r=3, padding=1, tile_m=4)
    rng = np.random.default_rng(512)
    w = rng.integers(-1, 2, spec.weight_shape()).astype(np.int8)
    x = rng.integers(-128, 128, spec.input_shape()).astype(np.int8)
    sys8 = rnsw.RnsSystem((251, 241, 239))
    with pytest.raises(rnsw.DynamicRangeExceeded):
        rnsw.winograd_layer_conv(spec, w, x, sys8)
    got = rnsw.winograd_layer_conv(spec, w, x, sys8, declared_bound=300_000)
    assert np.array_equal(got, oracle.direct_conv_c(x, w, 1))


def test_precomputed_filters_all_forms():
    rnsw = _rnsw()
    spec = rnsw.LayerSpec(h=12, w=12, c=3, k=4, r=3, padding=1, tile_m=4)
    w, x = _operands(spec, 4)
    system = rnsw.RnsSystem((251, 241, 239))
    mts = rnsw.reduce_for_system(rnsw.cached_transforms(4, 3), system)
    bank = rnsw.precompute_filter_transforms(w, mts)
    assert sorted(bank) == sorted(system.moduli) and bank[251].shape == (6, 6, 3, 4)
    ref_bank = O.filter_bank(w, {m: O.modular_matrices(4, 3, m) for m in system.moduli})
    for m in system.moduli:
        assert np.array_equal(bank[m], ref_bank[m])
    base = rnsw.winograd_layer_conv(spec, w, x, system, declared_bound=system.signed_bound)
    for filt in (bank, ref_bank, {m: v.astype(np.int16) for m, v in ref_bank.items()}):
        got = rnsw.winograd_layer_conv(spec, w, x, system, declared_bound=system.signed_bound, filters=filt)
        assert np.array_equal(got, base)
    with pytest.raises(rnsw.ShapeMismatch):
        rnsw.winograd_layer_conv(spec, w, x, system, declared_bound=system.signed_bound, filters={251: bank[251]})
    with pytest.raises(rnsw.ShapeMismatch):
        rnsw.winograd_layer_conv(spec, w, x, system, declared_bound=system.signed_bound,
                                 filters={m: f[:, :, :2] for m, f in ref_bank.items()})


def test_torch_operands_stay_on_device_and_timings():
    import torch

    rnsw = _rnsw()
    spec = rnsw.LayerSpec(h=28, w=28, c=32, k=32, r=3, padding=1, tile_m=14, batch=2)
    w, x = _operands(spec, 9)
    system = rnsw.RnsSystem((4001, 4331))
    t = rnsw.StageTimings()
    y = rnsw.winograd_layer_conv(spec, torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda(), system,
                                 declared_bound=system.signed_bound, timings=t)
    assert isinstance(y, torch.Tensor) and y.is_cuda and y.dtype == torch.int32
    assert t.input_transform > 0 and t.gemm > 0 and t.backward_transform > 0
    assert np.array_equal(y.cpu().numpy(), oracle.direct_conv_c(x, w, 1))


def test_errors_are_raised_before_device_work():
    rnsw = _rnsw()
    spec = rnsw.LayerSpec(h=8, w=8, c=2, k=2, r=3, padding=1, tile_m=4)
    w, x = _operands(spec, 1)
    sys8 = rnsw.RnsSystem((251, 241, 239))
    with pytest.raises(rnsw.ShapeMismatch):
        rnsw.winograd_layer_conv(spec, w, x[:, :, :5], sys8)
    with pytest.raises(rnsw.UnsupportedStride):
        rnsw.winograd_layer_conv(rnsw.LayerSpec(h=8, w=8, c=2, k=2, r=3, padding=1, stride=2, tile_m=4), w, x, sys8)
    with pytest.raises(rnsw.DeviceError):
        # F(21,5): tile side 25 is outside the device path (N <= 24)
        s18 = rnsw.LayerSpec(h=24, w=24, c=2, k=2, r=5, padding=2, tile_m=21)
        w18, x18 = _operands(s18, 2)
        rnsw.winograd_layer_conv(s18, w18, x18, rnsw.RnsSystem((4001, 4331)), declared_bound=1000)


@pytest.mark.parametrize("seed", range(16))
def test_random_geometry_sweep(seed):
    rnsw = _rnsw()
    rng = np.random.default_rng(100 + seed)
    r = int(rng.choice([3, 5]))
    tm = int(rng.choice([t for t in (2, 4, 6, 8, 10, 12, 14) if t + r - 1 <= 16]))
    mods = [(251, 241, 239), (4001, 4331), (253, 251, 247)][seed % 3]
    if tm + r - 1 > 12 and mods == (253, 251, 247):
        mods = (251, 241, 239)
    spec = rnsw.LayerSpec(h=int(rng.integers(r, 40)), w=int(rng.integers(r, 40)), c=int(rng.integers(1, 200)),
                          k=int(rng.integers(1, 150)), r=r, padding=int(rng.integers(0, r)), tile_m=tm,
                          batch=int(rng.integers(1, 4)))
    w, x = _operands(spec, seed, -20, 20)
    system = rnsw.RnsSystem(mods)
    got = rnsw.winograd_layer_conv(spec, w, x, system, declared_bound=system.signed_bound)
    assert np.array_equal(got, oracle.direct_conv_c(x, w, spec.padding))


SMALL_C = [
    # h, w, c, k, r, pad, batch, tile_m, moduli, layout -- C <= 4 runs the compact
    # transform + CUDA-core product path (csrc/smallc.cu)
    (224, 224, 3, 64, 3, 1, 1, 14, (4001, 4331), "nhwc"),   # VGG16 conv1_1
    (30, 26, 1, 5, 3, 1, 2, 8, (251, 241, 239), "nhwc"),     # K not a multiple of 8
    (17, 19, 2, 33, 5, 2, 3, 12, (4001, 4331), "nchw"),      # N = 16 with R = 5, NCHW
    (20, 20, 4, 16, 3, 0, 2, 2, (251, 241, 239, 233), "nhwc"),  # four residues
    (40, 40, 3, 130, 3, 1, 1, 6, (253, 251, 247), "nchw"),   # 3 residues, Kp = 144
]


@pytest.mark.parametrize("case", SMALL_C, ids=lambda c: "x".join(map(str, c[:8])) + c[9])
def test_small_channel_path(case):
    rnsw = _rnsw()
    h, w, c, k, r, pad, batch, tm, mods, layout = case
    spec = rnsw.LayerSpec(h=h, w=w, c=c, k=k, r=r, padding=pad, batch=batch, tile_m=tm)
    system = rnsw.RnsSystem(mods)
    wt, x = _operands(spec, c * 31 + k)
    want = O.winograd_layer(x, wt, pad, tm, mods)
    if layout == "nhwc":
        got = rnsw.winograd_layer_conv(spec, wt, x, system, declared_bound=system.signed_bound)
    else:
        got = rnsw.conv2d_rns(np.ascontiguousarray(x.transpose(0, 3, 1, 2)),
                              np.ascontiguousarray(wt.transpose(3, 2, 0, 1)), mods, tile_m=tm, padding=pad,
                              declared_bound=system.signed_bound)
        got = np.asarray(got).transpose(0, 2, 3, 1)
    assert np.array_equal(got, want)


def test_small_channel_wraps_like_the_reference():
    """A false declared bound wraps modulo D on the small-channel path too."""
    rnsw = _rnsw()
    spec = rnsw.LayerSpec(h=12, w=12, c=3, k=8, r=3, padding=1, tile_m=6)
    mods = (7, 11, 13)
    system = rnsw.RnsSystem(mods)
    wt, x = _operands(spec, 5)
    got = rnsw.winograd_layer_conv(spec, wt, x, system, declared_bound=10)
    assert np.array_equal(got, O.winograd_layer(x, wt, 1, 6, mods))


K1_STORES = [
    # (batch, side, c, k, r, tile_m, moduli, layout): the input transform's bulk
    # stores for several channel blocks, short tiles (N < 16) and NCHW input
    (2, 23, 200, 16, 3, 8, (251, 241, 239), "nhwc"),   # Cp = 256: 4 channel blocks, N = 10
    (3, 19, 40, 24, 5, 6, (4001, 4331), "nchw"),       # Cp = 64 with C = 40, N = 10, NCHW
    (1, 64, 32, 8, 3, 12, (4001, 4331), "nhwc"),       # Cp = 32 (box wider than the rows), N = 14
]


@pytest.mark.parametrize("case", K1_STORES, ids=lambda c: "c%d_n%d_%s" % (c[2], c[5] + c[4] - 1, c[7]))
def test_input_transform_bulk_store_layouts(case):
    rnsw = _rnsw()
    batch, side, c, k, r, tm, mods, layout = case
    spec = rnsw.LayerSpec(h=side, w=side, c=c, k=k, r=r, padding=r // 2, batch=batch, tile_m=tm)
    system = rnsw.RnsSystem(mods)
    wt, x = _operands(spec, side * c, -50, 50)
    want = oracle.direct_conv_c(x, wt, r // 2)
    if layout == "nhwc":
        got = rnsw.winograd_layer_conv(spec, wt, x, system, declared_bound=system.signed_bound)
    else:
        got = np.asarray(rnsw.conv2d_rns(np.ascontiguousarray(x.transpose(0, 3, 1, 2)),
                                         np.ascontiguousarray(wt.transpose(3, 2, 0, 1)), mods, tile_m=tm,
                                         padding=r // 2, declared_bound=system.signed_bound)).transpose(0, 2, 3, 1)
    assert np.array_equal(got, want)


GEMM_PATHS = [
    # (batch, side, c, k, tile_m, moduli): P = batch * ceil(side/tile_m)^2 tiles
    (3, 42, 64, 64, 14, (4001, 4331)),      # P = 27: one partial block, per-thread epilogue stores
    (16, 42, 64, 64, 14, (4001, 4331)),     # P = 144: 2 blocks, mostly dead -> per-thread stores
    (128, 28, 128, 256, 14, (4001, 4331)),  # P = 512: CTA pairs, 4 full blocks, bulk stores, num_kb = 2
    (72, 28, 256, 128, 14, (4001, 4331)),   # P = 288: odd block count (3) -> phantom partner block
    (64, 30, 32, 300, 10, (251, 241, 239)), # 8-bit: BN = 256 (per-thread stores), Kp = 304
    (64, 30, 96, 100, 10, (251, 241, 239)), # 8-bit: BN = 128 with bulk stores, Cp = 128
]


@pytest.mark.parametrize("case", GEMM_PATHS, ids=lambda c: "b%d_s%d_c%d_k%d" % c[:4])
def test_gemm_epilogue_and_pairing_paths(case):
    """Each GEMM variant (per-thread vs bulk-store epilogue, CTA pairs with an
    odd block count, 8-bit BN = 256) against the exact direct convolution."""
    rnsw = _rnsw()
    batch, side, c, k, tm, mods = case
    spec = rnsw.LayerSpec(h=side, w=side, c=c, k=k, r=3, padding=1, batch=batch, tile_m=tm)
    system = rnsw.RnsSystem(mods)
    wt, x = _operands(spec, batch + c, -40, 40)
    got = rnsw.winograd_layer_conv(spec, wt, x, system, declared_bound=system.signed_bound)
    assert np.array_equal(got, oracle.direct_conv_c(x, wt, 1))


DIRECT = [
    # b, h, w, c, k, r, pad, stride
    (1, 56, 56, 64, 64, 3, 1, 1),
    (2, 28, 28, 256, 96, 3, 1, 1),
    (3, 17, 23, 32, 40, 3, 1, 2),
    (1, 224, 224, 64, 64, 3, 1, 1),
    (2, 30, 30, 128, 300, 5, 2, 1),
    (1, 9, 9, 48, 8, 3, 0, 3),
    (4, 14, 14, 512, 512, 3, 1, 1),
]


@pytest.mark.parametrize("case", DIRECT, ids=lambda c: "x".join(map(str, c)))
def test_direct_conv_matches_oracle(case):
    rnsw = _rnsw()
    b, h, w, c, k, r, pad, stride = case
    spec = rnsw.LayerSpec(h=h, w=w, c=c, k=k, r=r, padding=pad, stride=stride, batch=b)
    wt, x = _operands(spec, h + c)
    got = rnsw.direct_conv(spec, wt, x)
    want = O.direct_conv(x, wt, pad) if stride == 1 else None
    if stride == 1:
        assert np.array_equal(got, want)
    else:
        full = oracle.direct_conv_c(x, wt, pad)
        assert np.array_equal(got, full[:, ::stride, ::stride][:, : spec.out_h, : spec.out_w])


def test_layer_conv_strided_uses_device_direct_conv():
    rnsw = _rnsw()
    spec = rnsw.LayerSpec(h=9, w=9, c=16, k=3, r=3, padding=1, stride=2, tile_m=4)
    wt, x = _operands(spec, 3)
    got = rnsw.layer_conv(spec, wt, x, rnsw.RnsSystem((251, 241, 239)))
    assert np.array_equal(got, oracle.direct_conv_c(x, wt, 1)[:, ::2, ::2])
    # C not a multiple of 16 computes too (rw/layer.py:402-403), channels
    # zero-padded on the device
    odd = rnsw.LayerSpec(h=9, w=9, c=2, k=3, r=3, padding=1, stride=2, tile_m=4)
    wb, xb = _operands(odd, 4)
    got = rnsw.layer_conv(odd, wb, xb, rnsw.RnsSystem((251, 241, 239)))
    assert np.array_equal(got, oracle.direct_conv_c(xb, wb, 1)[:, ::2, ::2])


def test_direct_conv_config5_digest():
    from golden_util import digests, sha
    from paper_2007_12216_b200 import workloads as W

    rnsw = _rnsw()
    w, x = W.config5_operands()
    spec = rnsw.LayerSpec(h=28, w=28, c=256, k=256, r=3, padding=1, batch=32)
    assert sha(rnsw.direct_conv(spec, w, x)) == digests()["cfg5/direct"]["y"]
