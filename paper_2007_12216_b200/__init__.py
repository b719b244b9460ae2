"""B200-native exact INT8 convolution by Winograd over a Residue Number System.

Drop-in for the layer-level hot path of the reference package ``rnswinograd``
(``winograd_layer_conv``, rw/layer.py:301-389): same entry points, argument
meaning and exception classes, with the arithmetic in hand-written sm_100a
CUDA kernels (tcgen05 kind::i8 tensor cores, TMA, TMEM) reached through the
C ABI in include/rnsw.h.  There is no CPU compute path.
"""

from .errors import (
    DeviceError,
    DynamicRangeExceeded,
    NotCoprime,
    OutOfRange,
    OverflowRisk,
    RnsError,
    ShapeMismatch,
    SystemMismatch,
    UnsupportedStride,
)
from .layer import (
    DirectWeights,
    FilterBank,
    LayerSpec,
    RangeReport,
    StageTimings,
    TilePlacement,
    conv2d_rns,
    count_operations,
    direct_conv,
    layer_conv,
    precompute_filter_transforms,
    precompute_filters_oihw,
    range_check,
    tile_decompose,
    winograd_layer_conv,
)
from .residue import RnsSystem, mod_inverse, mod_reduce
from .tensor_io import QTNS_MAGIC, QTNS_VERSION, read_tensor, write_tensor
from .tiles import rns_tile_conv, tile_conv_mod
from .transforms import (
    INF,
    ExactTransformSet,
    ModularTransformSet,
    cached_transforms,
    check_modulus_compatibility,
    default_points,
    derive_transforms,
    reduce_for_system,
    reduce_transforms_mod,
    vandermonde,
    vandermonde_inverse,
)

__version__ = "0.1.0"

__all__ = [
    "RnsError", "NotCoprime", "SystemMismatch", "OutOfRange", "DynamicRangeExceeded", "ShapeMismatch",
    "OverflowRisk", "UnsupportedStride", "DeviceError",
    "RnsSystem", "mod_reduce", "mod_inverse",
    "INF", "ExactTransformSet", "ModularTransformSet", "default_points", "vandermonde", "vandermonde_inverse",
    "derive_transforms", "cached_transforms", "check_modulus_compatibility", "reduce_transforms_mod",
    "reduce_for_system",
    "LayerSpec", "RangeReport", "StageTimings", "FilterBank", "TilePlacement", "range_check", "count_operations",
    "tile_decompose",
    "precompute_filter_transforms", "precompute_filters_oihw", "winograd_layer_conv", "layer_conv", "conv2d_rns",
    "direct_conv", "DirectWeights",
    "read_tensor", "write_tensor", "QTNS_MAGIC", "QTNS_VERSION", "tile_conv_mod", "rns_tile_conv",
    "__version__",
]
