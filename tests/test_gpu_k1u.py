"""The tcgen05 input transform (csrc/input_umma.cu: V = kron(BT, BT) d mod m
as one tensor-core GEMM per residue and position block, TMA patch boxes)
against the oracle's input stage (rw/kernel.py:44-47 via oracle/ref_port.py)
and end to end.  It serves NHWC layers with C = 64 (tile pairs) or
C % 128 == 0 on every tensor-core plan; other shapes keep the mma.sync kernel
(covered by test_gpu_layer.py)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from oracle import ref_port as O

pytestmark = pytest.mark.gpu

SYS8 = (251, 241, 239)
SYS16 = (4001, 4331)

# (h, w, c, batch, tile_m, r, pad, moduli): N = tile_m + r - 1 from 6 to 16,
# one and two 128-position blocks, odd tile counts (the last tile pair has
# one real tile), ragged edges, the full int8 range
STAGE_CASES = [
    (30, 30, 64, 1, 14, 3, 1, SYS16),    # N=16, tile pairs, P = 9 (odd)
    (28, 17, 128, 2, 14, 3, 1, SYS16),   # N=16, one tile x 128 channels
    (16, 16, 256, 1, 14, 3, 1, SYS16),   # two channel blocks
    (21, 19, 64, 2, 8, 3, 1, SYS8),      # N=10, 8-bit, 1 position block
    (13, 13, 128, 1, 6, 3, 1, SYS8),     # N=8
    (25, 25, 64, 1, 12, 3, 1, SYS8),     # N=14, 8-bit, 2 position blocks (K = 196 -> 224)
    (20, 20, 64, 1, 6, 3, 1, SYS16),     # N=8, 16-bit
    (11, 11, 128, 3, 4, 3, 0, (253, 251, 247)),  # N=6, no padding
    (19, 23, 64, 1, 8, 5, 2, SYS8),      # 5x5 filter: N=12
]


def _ids(c):
    return f"{c[0]}x{c[1]}x{c[2]}-b{c[3]}-F{c[4]},{c[5]}-{len(c[7])}res"


@pytest.mark.parametrize("case", STAGE_CASES, ids=_ids)
def test_input_transform_matches_oracle(case):
    import torch

    import paper_2007_12216_b200 as rnsw
    from paper_2007_12216_b200 import stages

    h, w, c, b, tm, r, pad, mods = case
    rng = np.random.default_rng(h * 131 + c)
    x = rng.integers(-128, 128, (b, h, w, c)).astype(np.int8)
    x.reshape(-1)[:7] = [-128, 127, -128, 127, 0, -1, 1]
    system = rnsw.RnsSystem(mods)
    _, vres, p = stages.input_transform(x, tm, r, system, pad)
    torch.cuda.synchronize()
    patches, _ = O.patches_of(x, tm, r, pad)
    for m in mods:
        _, _, bt = O.modular_matrices(tm, r, m)
        assert np.array_equal(vres[m].cpu().numpy(), O.input_stage(patches, bt, m)), f"mod {m}"


@pytest.mark.parametrize("case", STAGE_CASES, ids=_ids)
def test_layer_with_umma_input_transform(case):
    import paper_2007_12216_b200 as rnsw

    h, w, c, b, tm, r, pad, mods = case
    rng = np.random.default_rng(h * 7 + c)
    k = 48
    wt = rng.integers(-128, 128, (r, r, c, k)).astype(np.int8)
    x = rng.integers(-128, 128, (b, h, w, c)).astype(np.int8)
    system = rnsw.RnsSystem(mods)
    spec = rnsw.LayerSpec(h=h, w=w, c=c, k=k, r=r, padding=pad, batch=b, tile_m=tm)
    got = rnsw.winograd_layer_conv(spec, wt, x, system, declared_bound=system.signed_bound)
    assert np.array_equal(got, O.winograd_layer(x, wt, pad, tm, mods))


def test_vgg_shapes_activations_in_range():
    """conv1_2 / conv2_1 / conv3_1 shapes (C = 64, 64, 128) at batch 3 with
    [0, 127] activations: exact against direct conv."""
    import paper_2007_12216_b200 as rnsw

    rng = np.random.default_rng(99)
    for side, c, k in [(224, 64, 64), (112, 64, 128), (56, 128, 256)]:
        x = rng.integers(0, 128, (3, side, side, c)).astype(np.int8)
        wt = np.clip(np.rint(rng.normal(0, 20, (3, 3, c, k))), -127, 127).astype(np.int8)
        spec = rnsw.LayerSpec(h=side, w=side, c=c, k=k, r=3, padding=1, batch=3, tile_m=14)
        system = rnsw.RnsSystem(SYS16)
        got = rnsw.winograd_layer_conv(spec, wt, x, system, declared_bound=system.signed_bound)
        assert np.array_equal(got, oracle.direct_conv_c(x, wt, 1)), (side, c, k)


@pytest.mark.skipif(os.environ.get("RNSW_K1_MMA_SYNC") is not None, reason="already the alternate path")
def test_mma_sync_input_transform_still_matches():
    """RNSW_K1_MMA_SYNC=1 keeps the mma.sync kernel for these shapes: rerun the
    stage checks on it in a subprocess (the switch is read once per process)."""
    env = dict(os.environ, RNSW_K1_MMA_SYNC="1")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_k1u.py"), "-k", "input_transform_matches"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.skipif(os.environ.get("RNSW_K1_PAIR") is not None, reason="already the alternate path")
def test_cta_pair_input_transform_still_matches():
    """RNSW_K1_PAIR=1 runs K1 as 2-CTA clusters (cta_group::2 MMAs of M = 256,
    the patch split by channels between the pair) where a residue has two
    128-position blocks: rerun the stage and whole-layer checks on it."""
    env = dict(os.environ, RNSW_K1_PAIR="1")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_k1u.py"), "-k", "not still"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
