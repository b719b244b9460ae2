"""GPU parity: the sm_100a path against the CPU oracle, stage by stage and
end to end.  The oracle (oracle/ref_port.py) is pinned to the reference by
tests/test_oracle.py; ``direct_conv`` is the exact convolution."""

import numpy as np
import pytest

import oracle
from oracle import ref_port as O

pytestmark = pytest.mark.gpu

SYS8 = (251, 241, 239)
SYS16 = (4001, 4331)

# (h, w, c, k, r, pad, batch, tile_m, moduli): the reference's FAST_CASES
# geometries (t/test_layer.py:161-168) plus one config-shaped layer each.
CASES = [
    (8, 8, 3, 5, 3, 1, 2, 4, SYS8),
    (16, 16, 4, 3, 5, 2, 1, 12, SYS16),
    (30, 30, 7, 2, 3, 0, 1, 14, SYS8),
    (28, 28, 32, 16, 3, 1, 1, 14, SYS8),
    (6, 10, 2, 2, 3, 1, 1, 2, (253, 251, 247)),
    (56, 56, 64, 64, 3, 1, 1, 8, SYS8),
    (20, 20, 96, 80, 3, 1, 2, 6, SYS16),
    (14, 14, 160, 40, 3, 1, 1, 14, SYS16),
    (17, 13, 33, 17, 5, 2, 3, 8, SYS8),
    (9, 9, 5, 3, 3, 1, 1, 4, (7, 11, 13)),
    (12, 12, 130, 300, 3, 1, 1, 10, (251, 4001)),
]


def _rnsw():
    import paper_2007_12216_b200 as rnsw

    return rnsw


def _operands(h, w, c, k, r, batch, seed):
    rng = np.random.default_rng(seed)
    wt = rng.integers(-128, 128, (r, r, c, k)).astype(np.int8)
    x = rng.integers(-128, 128, (batch, h, w, c)).astype(np.int8)
    return wt, x


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[:8])) + f"-{len(c[8])}res")
def test_layer_matches_oracle_and_direct(case):
    rnsw = _rnsw()
    h, w, c, k, r, pad, batch, tm, mods = case
    wt, x = _operands(h, w, c, k, r, batch, h * 1000 + c)
    spec = rnsw.LayerSpec(h=h, w=w, c=c, k=k, r=r, padding=pad, batch=batch, tile_m=tm)
    system = rnsw.RnsSystem(mods)
    got = rnsw.winograd_layer_conv(spec, wt, x, system, declared_bound=system.signed_bound)
    assert got.dtype == np.int32 and got.shape == (batch, spec.out_h, spec.out_w, k)
    ref = O.winograd_layer(x, wt, pad, tm, mods)
    assert np.array_equal(got, ref)
    direct = oracle.direct_conv_c(x, wt, pad)
    if np.abs(direct.astype(np.int64)).max() <= system.signed_bound:
        assert np.array_equal(got, direct)


@pytest.mark.parametrize("case", CASES[:6] + CASES[9:], ids=lambda c: "x".join(map(str, c[:8])))
def test_stages_match_oracle(case):
    import torch

    rnsw = _rnsw()
    from paper_2007_12216_b200 import stages

    h, w, c, k, r, pad, batch, tm, mods = case
    wt, x = _operands(h, w, c, k, r, batch, 7 + c)
    system = rnsw.RnsSystem(mods)
    mats = {m: O.modular_matrices(tm, r, m) for m in mods}
    patches, _ = O.patches_of(x, tm, r, pad)
    vbuf, vres, p = stages.input_transform(x, tm, r, system, pad)
    bank = rnsw.precompute_filter_transforms(wt, rnsw.reduce_for_system(rnsw.cached_transforms(tm, r), system))
    ubank = O.filter_bank(wt, mats)
    mw, accs = stages.winograd_gemm(vbuf, bank.data, tm, r, system, p, c, k)
    ys = stages.output_residues(mw, tm, r, system, p, k)
    torch.cuda.synchronize()
    for m in mods:
        at, _, bt = mats[m]
        v_ref = O.input_stage(patches, bt, m)
        assert np.array_equal(vres[m].cpu().numpy(), v_ref), f"input transform mod {m}"
        assert np.array_equal(bank[m], ubank[m]), f"filter transform mod {m}"
        acc_ref = O.gemm_stage(v_ref, ubank[m], m)
        assert np.array_equal(accs[m].cpu().numpy().astype(np.int32), acc_ref), f"gemm mod {m}"
        y_ref = O.output_stage(acc_ref, at, m)
        assert np.array_equal(ys[m].cpu().numpy(), y_ref), f"backward transform mod {m}"


@pytest.mark.parametrize("mods", [SYS8, SYS16, (253, 251, 247), (7, 11, 13), (251, 4001)])
def test_mrc_matches_oracle(mods):
    from paper_2007_12216_b200 import stages

    rnsw = _rnsw()
    system = rnsw.RnsSystem(mods)
    rng = np.random.default_rng(len(mods))
    vals = rng.integers(-system.signed_bound, system.signed_bound + 1, 5000, dtype=np.int64)
    vals[:4] = [0, system.signed_bound, -system.signed_bound, 1]
    res = np.stack([O.fold(vals.copy(), m) for m in mods]).astype(np.int16)
    got = stages.mrc_reconstruct(res, 4, 3, system).cpu().numpy()
    assert np.array_equal(got, O.mrc(list(res), mods))
    assert np.array_equal(got, vals)
