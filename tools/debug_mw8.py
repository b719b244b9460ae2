"""Check the tcgen05 output transform (rnsw_output_transform_mw8) on synthetic
Mw8 input against numpy: Y = AT M AT^T mod m per residue, MRC, crop; prints
the mismatch pattern per tile row/column/channel (a debugging aid; the
pytest version is tests/test_gpu_mw8.py).

usage: python tools/debug_mw8.py [mode]   mode: rand | delta I J | const
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2007_12216_b200 as rnsw
from paper_2007_12216_b200 import _native
from paper_2007_12216_b200.layer import _stream_ptr, plan_for

mods = (4001, 4331)
ts = rnsw.cached_transforms(14, 3)
system = rnsw.RnsSystem(mods)
plan = plan_for(ts, system)
l = _native.lib()
assert l.rnsw_mw8_supported(plan.handle) == 1
B, H, K = 1, 28, 32
P = B * ((H + 13) // 14) ** 2
Kp = (K + 15) // 16 * 16
rng = np.random.default_rng(1)
mode = sys.argv[1] if len(sys.argv) > 1 else "rand"
mat = np.zeros((2, P, 256, K), np.int64)
if mode == "rand":
    for r, m in enumerate(mods):
        mat[r] = rng.integers(0, m, (P, 256, K))
elif mode == "delta":
    i, j = int(sys.argv[2]), int(sys.argv[3])
    mat[:, :, i * 16 + j, :] = 1
elif mode == "const":
    mat[:] = 1
num_pb = (P + 127) // 128
mw8 = np.zeros((num_pb, 2, 2, 256, 128, Kp), np.uint8)
for p in range(P):
    for r in range(2):
        mw8[p >> 7, r, 0, :, p & 127, :K] = mat[r, p] & 255
        mw8[p >> 7, r, 1, :, p & 127, :K] = mat[r, p] >> 8
dev = torch.from_numpy(mw8.reshape(-1)).cuda()
y = torch.zeros((B, H, H, K), dtype=torch.int32, device="cuda")
_native.check(l.rnsw_output_transform_mw8(plan.handle, _native.c_void_p(dev.data_ptr()), B, H, H, K, 1, 0,
                                          _native.c_void_p(y.data_ptr()), _stream_ptr()))
torch.cuda.synchronize()
got = y.cpu().numpy()

# numpy expectation
mts = rnsw.transforms.reduce_for_system(ts, system)
yr = []
for r, m in enumerate(mods):
    AT = mts[r].at.astype(np.int64)
    M = mat[r].reshape(P, 16, 16, K)
    Y = np.einsum("ai,pijk,bj->pabk", AT, M, AT) % m
    yr.append(Y)
m0, m1 = mods
inv = pow(m0, -1, m1)
d1 = ((yr[1] - yr[0]) * inv) % m1
x = yr[0] + m0 * d1
D = m0 * m1
x = np.where(x > (D - 1) // 2, x - D, x)
th = (H + 13) // 14
want = np.zeros_like(got)
for p in range(P):
    b, rem = divmod(p, th * th)
    ti, tj = divmod(rem, th)
    for a in range(14):
        for bb in range(14):
            ho, wo = ti * 14 + a, tj * 14 + bb
            if ho < H and wo < H:
                want[b, ho, wo, :] = x[p, a, bb, :]
bad = got != want
print("mismatches", bad.sum(), "of", bad.size)
if bad.any():
    idx = np.argwhere(bad)
    print("first", idx[:10].tolist())
    print("got", got[tuple(idx[0])], "want", want[tuple(idx[0])])
    # pattern per (a, b) inside tile 0 and per channel
    t0 = bad[0, :14, :14, :]
    print("bad per a", t0.sum(axis=(1, 2)).tolist())
    print("bad per b", t0.sum(axis=(0, 2)).tolist())
    print("bad per k", t0.sum(axis=(0, 1)).tolist())
    print("got tile0 k0\n", got[0, :14, :14, 0])
    print("want tile0 k0\n", want[0, :14, :14, 0])
