"""Run one VGG16 layer through rnsw_conv_forward_requant a few times (profiling driver).

usage: python tools/one_layer_fused.py <layer-name> <batch> [iters]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2007_12216_b200 import _native, workloads as W
from paper_2007_12216_b200.vgg import VGG16Rns

name = sys.argv[1] if len(sys.argv) > 1 else "conv1_2"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
names = [l[0] for l in W.VGG16_LAYERS]
i = names.index(name)
_, side, c, k, pool = W.VGG16_LAYERS[i]
net = VGG16Rns()
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.integers(0, 128, (B, side, side, c), dtype=np.int8)).cuda()
bufs = net._alloc(B)
oside = side // 2 if pool else side
out = torch.empty((B, oside, oside, k), dtype=torch.int8, device="cuda")
l = _native.lib()
vp = _native.c_void_p
s = _native.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(iters):
    _native.check(l.rnsw_conv_forward_requant(net.plan.handle, vp(x.data_ptr()), B, side, side, c, k, 1,
                                              vp(net.banks[i].data.data_ptr()), net.cfg.shifts[i], 1 if pool else 0,
                                              vp(out.data_ptr()), vp(bufs["ws"].data_ptr()), bufs["ws"].numel(), s))
torch.cuda.synchronize()
print("ok", name, B)
