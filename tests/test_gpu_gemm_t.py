"""The small-P GEMM (csrc/gemm_t.cu: output channels on the MMA rows, tiles on
the columns, only the u limb planes of the filter bank, three accumulators)
that whole-layer calls with 16-bit residues and at most 48 tiles (80 for C >= 512) take
(rw/layer.py:285-291 semantics): end to end against the exact direct
convolution, including tile counts that are not multiples of 16, K that is
not a multiple of 128 (the last channel block is partly outside Kp), several
128-channel blocks, full-range int8 operands, and the regular GEMM forced
for the same shapes in a subprocess."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

SYS16 = (4001, 4331)

# (h, w, c, k, batch, tile_m): P = batch * ceil(h/m) * ceil(w/m); both GEMMs run every case (forced below)
CASES = [
    (14, 14, 128, 64, 1, 14),    # P = 1
    (28, 28, 256, 96, 3, 14),    # P = 12, K = 96 (one partial channel block)
    (42, 29, 128, 200, 2, 14),   # P = 18 -> N = 32, K = 200 (two blocks, the second partial)
    (56, 56, 128, 48, 2, 14),    # P = 32
    (30, 30, 384, 144, 5, 14),   # P = 45 -> N = 48, C = 384 (three 128-channel chunks)
    (24, 24, 128, 128, 4, 10),   # F(10,3): N = 12 (144 positions), P = 36
    (28, 28, 128, 128, 16, 14),  # P = 64
    (28, 28, 256, 160, 20, 14),  # P = 80, K = 160
    (28, 28, 128, 128, 23, 14),  # P = 92 -> N = 96 (single-buffered accumulators)
    (28, 28, 512, 256, 32, 14),  # P = 128: the deep VGG16 layers at batch 32
    (14, 14, 512, 128, 64, 14),  # P = 64, C = 512: small-P GEMM by default (conv5 at batch 64)
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}x{c[1]}x{c[2]}->{c[3]}-b{c[4]}-F{c[5]}")
def test_small_p_layer_matches_direct_conv(case):
    import paper_2007_12216_b200 as rnsw

    h, w, c, k, b, tm = case
    rng = np.random.default_rng(hash(case) & 0xFFFFFFFF)
    x = rng.integers(-128, 128, (b, h, w, c), dtype=np.int8)
    wt = rng.integers(-128, 128, (3, 3, c, k), dtype=np.int8)
    spec = rnsw.LayerSpec(h=h, w=w, c=c, k=k, r=3, padding=1, batch=b, tile_m=tm)
    system = rnsw.RnsSystem(SYS16)
    got = rnsw.winograd_layer_conv(spec, wt, x, system, declared_bound=system.signed_bound)
    want = oracle.direct_conv_c(x, wt, 1)
    # |y| <= 9 c 128^2 may exceed (D - 1) / 2: compare modulo D, symmetric
    d = int(np.prod(SYS16))
    diff = (got.astype(np.int64) - want.astype(np.int64)) % d
    assert np.all(diff == 0), case
    small = np.abs(want.astype(np.int64)) <= system.signed_bound
    assert np.array_equal(got[small], want[small])


@pytest.mark.skipif(os.environ.get("RNSW_GEMM_T") is not None, reason="already forced")
@pytest.mark.parametrize("max_p", ["0", "128"])
def test_forced_gemm_choice_for_the_same_shapes(max_p):
    """RNSW_GEMM_T=0: the tile-row GEMM for every P; =128: the small-P GEMM for
    every case above (N up to 128); the same checks must hold."""
    env = dict(os.environ, RNSW_GEMM_T=max_p)
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_gemm_t.py"), "-k", "matches_direct"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
