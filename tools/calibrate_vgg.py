"""One-off calibration of VGG16_SHIFTS (paper_2007_12216_b200/workloads.py).

For each layer pick the smallest shift s with percentile_99.5(relu(y)) >> s
<= 127 on the seed-2020 image 0, propagating the requantised activations.
Uses the C direct-conv oracle (exact int32).  Prints the table to freeze.
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
from oracle.vgg_ref import requant_pool  # noqa: E402
from paper_2007_12216_b200 import workloads as W  # noqa: E402

ws = W.vgg16_weights()
x = W.vgg16_images(1)
shifts, maxes = [], []
for (name, side, c, k, pool), w in zip(W.VGG16_LAYERS, ws):
    y = oracle.direct_conv_c(x, w, 1)
    pos = y[y > 0]
    q = np.percentile(pos, 99.5) if pos.size else 1
    s = max(0, int(np.ceil(np.log2(max(q, 1) / 127.0))))
    shifts.append(s)
    maxes.append(int(np.abs(y).max()))
    x = requant_pool(y, s, pool)
    print(name, "max|y|", maxes[-1], "shift", s, "act mean", float(x.mean()))
print("VGG16_SHIFTS =", tuple(shifts))
print("bounds", W.vgg16_bounds(ws))
