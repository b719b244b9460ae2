"""Host-side logic of the product (no GPU): exact transform construction,
residue systems, range checks, argument validation and exception order,
all pinned to the reference's golden values and known answers."""
import math

import numpy as np
import pytest

import paper_2007_12216_b200 as rnsw
from paper_2007_12216_b200 import errors, residue, transforms
from paper_2007_12216_b200.layer import LayerSpec, range_check
from golden_util import scalars, transforms as golden_transforms


def test_modular_transforms_match_reference_golden():
    for key, ent in golden_transforms().items():
        fm, mod = key.split("/")
        m_out, r = (int(v) for v in fm[1:].split("x"))
        ts = transforms.cached_transforms(m_out, r)
        assert transforms.check_modulus_compatibility(ts, int(mod)) == ent["compatible"], key
        if ent["compatible"]:
            mt = transforms.reduce_transforms_mod(ts, int(mod))
            assert mt.at.tolist() == ent["at"] and mt.g.tolist() == ent["g"] and mt.bt.tolist() == ent["bt"]
            assert str(mt.at.dtype) == ent["dtype"] and not mt.at.flags.writeable
        else:
            with pytest.raises(errors.NotCoprime):
                transforms.reduce_transforms_mod(ts, int(mod))


def test_incompatible_moduli_at_large_tiles():
    # 253 = 11*23 fails from N = 13 on, 247 = 13*19 from N = 15 (t/test_transforms.py:249-262)
    assert transforms.check_modulus_compatibility(transforms.cached_transforms(10, 3), 253)
    assert not transforms.check_modulus_compatibility(transforms.cached_transforms(12, 3), 253)
    assert transforms.check_modulus_compatibility(transforms.cached_transforms(12, 3), 247)
    assert not transforms.check_modulus_compatibility(transforms.cached_transforms(14, 3), 247)


def test_vandermonde_inverse_is_exact():
    for n in range(2, 12):
        pts = transforms.default_points(n)
        v, vi = transforms.vandermonde(pts), transforms.vandermonde_inverse(pts)
        for i in range(n):
            for j in range(n):
                assert sum(v[i][k] * vi[k][j] for k in range(n)) == (1 if i == j else 0)


def test_winograd_identity_1d_exact():
    # y = AT ((G g) * (BT d)) equals direct correlation, exactly, for random integers
    rng = np.random.default_rng(1)
    for m_out, r in [(2, 3), (6, 3), (8, 5), (14, 3)]:
        ts = transforms.cached_transforms(m_out, r)
        n = ts.n
        g = [int(v) for v in rng.integers(-9, 10, r)]
        d = [int(v) for v in rng.integers(-9, 10, n)]
        u = [sum(ts.g[i][k] * g[k] for k in range(r)) for i in range(n)]
        v = [sum(ts.bt[i][k] * d[k] for k in range(n)) for i in range(n)]
        y = [sum(ts.at[i][k] * u[k] * v[k] for k in range(n)) for i in range(m_out)]
        want = [sum(g[k] * d[i + k] for k in range(r)) for i in range(m_out)]
        assert y == want


def test_system_constants_match_reference():
    for key, ent in scalars().items():
        if not key[0].isdigit():
            continue
        mods = tuple(int(v) for v in key.split("x"))
        s = residue.RnsSystem(mods)
        assert s.signed_bound == ent["signed_bound"] and s.dynamic_range == ent["dynamic_range"]
        assert s._mrc_inv == ent["mrc_inv"]
        t = s.mrc_table()
        for j in range(len(mods)):
            for i in range(j):
                assert (mods[i] * int(t[j, i])) % mods[j] == 1


def test_signed_bounds_known_answers():
    # t/test_acceptance.py:151-157
    assert residue.RnsSystem((253, 251, 247)).signed_bound == 7_842_620
    assert residue.RnsSystem((251, 241, 239)).signed_bound == 7_228_674
    assert residue.RnsSystem((4001, 4331)).signed_bound == 8_664_165


def test_mod_inverse_known_answers():
    # t/test_residue.py:67-71
    for m, v in scalars()["mod_inverse_14400"].items():
        assert residue.mod_inverse(14400, int(m)) == v
    assert [residue.mod_inverse(14400, m) for m in (253, 251, 247)] == [12, 27, -10]


def test_scalar_reconstruct_round_trip():
    s = residue.RnsSystem((7, 11, 13))
    for x in range(-s.signed_bound, s.signed_bound + 1):
        assert s.reconstruct(s.encode(x)) == x
    with pytest.raises(errors.OutOfRange):
        s.encode(s.signed_bound + 1)


@pytest.mark.parametrize("bad", [(6, 7), (3, 9), (251, 251), (2,), (32769,), ()])
def test_system_rejects_bad_moduli(bad):
    with pytest.raises((ValueError, errors.NotCoprime)):
        residue.RnsSystem(bad)


def test_range_check_semantics():
    # rw/layer.py:191-208; messages of t/test_cli.py:152-166 use these numbers
    spec = LayerSpec(h=56, w=56, c=512, k=4, r=3, padding=1, tile_m=8)
    rep = range_check(spec, residue.RnsSystem((251, 241, 239)))
    assert rep.static_bound == 9 * 512 * 127 * 127 == 74_322_432 and not rep.fits
    assert rep.signed_bound == 7_228_674
    rep = range_check(spec, residue.RnsSystem((251, 241, 239)), declared_bound=300_000)
    assert rep.fits and rep.bound == 300_000
    cfg1 = LayerSpec(h=56, w=56, c=64, k=64, r=3, padding=1, tile_m=8)
    assert range_check(cfg1, residue.RnsSystem((251, 241, 239))).static_bound == 9_290_304


def test_layer_spec_validation_mirrors_reference():
    spec = LayerSpec(h=224, w=224, c=3, k=64, r=3, padding=1)
    assert (spec.out_h, spec.out_w) == (224, 224)
    spec = LayerSpec(h=7, w=9, c=1, k=1, r=3, padding=0, stride=2)
    assert (spec.out_h, spec.out_w) == (3, 4)
    for kw in (dict(h=0), dict(c=-1), dict(padding=-1), dict(tile_m=0), dict(h=1, w=1, r=3)):
        base = dict(h=8, w=8, c=2, k=2, r=3)
        base.update(kw)
        with pytest.raises(ValueError):
            LayerSpec(**base)


def _operands(spec, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.integers(-128, 128, spec.weight_shape()).astype(np.int8),
            rng.integers(-128, 128, spec.input_shape()).astype(np.int8))


def test_preflight_errors_before_device_work():
    """Checks run on the host in the reference's order (rw/layer.py:321-338)
    and raise before the GPU is touched, so they hold on a CPU-only host."""
    sys8 = rnsw.RnsSystem((251, 241, 239))
    spec = LayerSpec(h=8, w=8, c=2, k=2, r=3, padding=1, tile_m=4)
    w, x = _operands(spec)
    with pytest.raises(errors.ShapeMismatch):
        rnsw.winograd_layer_conv(spec, w[:, :, :1], x, sys8)
    with pytest.raises(errors.ShapeMismatch):
        rnsw.winograd_layer_conv(spec, w, x[:, :4], sys8)
    with pytest.raises(errors.ShapeMismatch):
        rnsw.winograd_layer_conv(spec, w.astype(np.int16), x, sys8)
    strided = LayerSpec(h=8, w=8, c=2, k=2, r=3, padding=1, stride=2, tile_m=4)
    with pytest.raises(errors.UnsupportedStride):
        rnsw.winograd_layer_conv(strided, w, x, sys8)
    # (layer_conv with stride != 1 computes on the device direct conv for every
    # C, like the reference's rw/layer.py:402-403: covered by the GPU tests)
    with pytest.raises(ValueError):
        rnsw.winograd_layer_conv(LayerSpec(h=8, w=8, c=2, k=2, r=3, padding=1), w, x, sys8)
    big = LayerSpec(h=8, w=8, c=512, k=2, r=3, padding=1, tile_m=4)
    wb, xb = _operands(big)
    with pytest.raises(errors.DynamicRangeExceeded):
        rnsw.winograd_layer_conv(big, wb, xb, sys8)
    with pytest.raises(errors.ShapeMismatch):
        rnsw.winograd_layer_conv(spec, w, x, sys8, declared_bound=1000,
                                 transform_set=transforms.cached_transforms(2, 3))
    # 253 = 11 * 23 cannot carry F(12,3) (N = 14)
    t12 = LayerSpec(h=16, w=16, c=2, k=2, r=3, padding=1, tile_m=12)
    w12, x12 = _operands(t12)
    with pytest.raises(errors.NotCoprime):
        rnsw.winograd_layer_conv(t12, w12, x12, rnsw.RnsSystem((253, 251, 247)), declared_bound=1000)


def test_count_operations_model():
    spec = LayerSpec(h=224, w=224, c=64, k=64, r=3, padding=1, tile_m=14)
    oc = rnsw.count_operations(spec, rnsw.RnsSystem((4001, 4331)))
    assert oc.tiles == 256
    assert oc.direct_mults == 224 * 224 * 64 * 64 * 9
    assert oc.winograd_mults == 256 * 256 * 64 * 64 * 2
    assert float(oc.reduction_ratio) == pytest.approx(14 * 14 * 9 / (16 * 16 * 2))


def test_limb_planes():
    assert [residue.planes_for_modulus(m) for m in (7, 251, 253, 4001, 32767)] == [1, 1, 1, 2, 2]


def test_error_code_mapping():
    for code, exc in [(2, errors.ShapeMismatch), (3, errors.UnsupportedStride), (4, errors.DynamicRangeExceeded),
                      (5, errors.NotCoprime), (6, errors.OverflowRisk), (7, errors.SystemMismatch),
                      (8, errors.DeviceError), (1, ValueError)]:
        with pytest.raises(exc):
            errors.raise_for(code, "x")
    errors.raise_for(0, "ok")
