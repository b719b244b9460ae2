"""ORACLE -- test infrastructure only.

CPU restatement of the VGG16 inter-layer glue the GPU stack applies
(relu, >> shift, clip to [0,127], 2x2 max-pool with floor) and of the whole
stack on top of the exact C direct convolution.  The glue is not part of the
reference package (SPEC.md:443 non-goals); BASELINE.json configs 2/4 define
it, and paper_2007_12216_b200/workloads.py freezes the shift table.
"""

from __future__ import annotations

import numpy as np

from . import direct_conv_c


def requant_pool(y: np.ndarray, shift: int, pool: bool) -> np.ndarray:
    v = np.clip(np.maximum(y, 0) >> shift, 0, 127).astype(np.int8)
    if pool:
        b, h, w, c = v.shape
        v = v[:, : h // 2 * 2, : w // 2 * 2].reshape(b, h // 2, 2, w // 2, 2, c).max(axis=(2, 4))
    return np.ascontiguousarray(v)


def vgg16_stack(x: np.ndarray, weights, layers, shifts, keep_int32: bool = False):
    """Exact stack: returns the final int8 map (and every layer's int32 output)."""
    outs = []
    for (name, side, c, k, pool), w, s in zip(layers, weights, shifts):
        y = direct_conv_c(x, w, 1)
        if keep_int32:
            outs.append(y)
        x = requant_pool(y, s, pool)
    return (x, outs) if keep_int32 else x
