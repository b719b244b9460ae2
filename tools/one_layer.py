"""Run one VGG16-shaped RNS-Winograd layer a few times (profiling driver).

usage: python tools/one_layer.py <layer-name> <batch> [iters]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2007_12216_b200 as rnsw
from paper_2007_12216_b200 import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "conv1_2"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
layer = {l[0]: l for l in W.VGG16_LAYERS}[name]
_, side, c, k, _ = layer
idx = [l[0] for l in W.VGG16_LAYERS].index(name)
w = W.vgg16_weights()[idx]
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.integers(0, 128, (B, side, side, c), dtype=np.int8)).cuda()
spec = rnsw.LayerSpec(h=side, w=side, c=c, k=k, r=3, padding=1, batch=B, tile_m=14)
system = rnsw.RnsSystem((4001, 4331))
bank = rnsw.precompute_filter_transforms(w, rnsw.reduce_for_system(rnsw.cached_transforms(14, 3), system))
bound = W.vgg16_bounds([w])[0]
for _ in range(iters):
    y = rnsw.winograd_layer_conv(spec, torch.from_numpy(w).cuda(), x, system, declared_bound=bound, filters=bank)
torch.cuda.synchronize()
print("ok", name, B, tuple(y.shape))
