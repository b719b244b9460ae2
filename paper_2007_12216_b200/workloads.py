"""Seeded synthetic workloads for BASELINE.json's five configs.

The reference's CLI derives independent PCG64 streams from
``SeedSequence([seed, label])`` with string labels folded to ints
(rw/cli.py:82-94) and generates weights before activations per layer
(rw/cli.py:439-441); the same convention is used here so CPU oracle and GPU
see byte-identical int8 tensors.  Layouts are the reference's: activations
NHWC (B,H,W,C), weights (R,R,C,K).  No dataset or checkpoint is involved:
ImageNet and pretrained VGG16 are replaced by seeded draws with the shapes
and value distributions BASELINE.json states.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DEFAULT_SEED = 2020  # rw/cli.py:30


def make_rng(*entropy) -> np.random.Generator:
    """rw/cli.py:82-94: string items fold to int.from_bytes(...) % 2**64, i.e.
    only their first 8 bytes count -- labels must differ there (or carry an
    int item) to give independent streams."""
    words = []
    for item in entropy:
        if isinstance(item, str):
            words.append(int.from_bytes(item.encode(), "little") % (1 << 64))
        else:
            words.append(int(item) % (1 << 64))
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(words)))


def uniform_int8(rng, shape, lo: int, hi: int) -> np.ndarray:
    """Integers uniform in [lo, hi] inclusive."""
    return rng.integers(lo, hi + 1, size=shape, dtype=np.int8)


def gaussian_int8(rng, shape, sigma: float = 20.0) -> np.ndarray:
    """round(N(0, sigma^2)) clipped to [-127, 127]."""
    return np.clip(np.rint(rng.normal(0.0, sigma, size=shape)), -127, 127).astype(np.int8)


def weight_bound(w: np.ndarray, xmax: int) -> int:
    """Sound bound on |y|: max over output channels of sum|w| * max|x|."""
    return int(np.abs(w.astype(np.int64)).reshape(-1, w.shape[-1]).sum(axis=0).max()) * int(xmax)


@dataclass(frozen=True)
class LayerCase:
    name: str
    batch: int
    h: int
    w: int
    c: int
    k: int
    r: int
    pad: int
    tile_m: int
    moduli: tuple
    declared_bound: int | None = None

    @property
    def out_h(self) -> int:
        return self.h + 2 * self.pad - self.r + 1

    @property
    def out_w(self) -> int:
        return self.w + 2 * self.pad - self.r + 1

    def direct_ops(self) -> int:
        """Direct-conv-equivalent integer ops: 2 * B * Ho * Wo * C * K * R^2."""
        return 2 * self.batch * self.out_h * self.out_w * self.c * self.k * self.r * self.r


SYS8 = (251, 241, 239)
SYS8B = (253, 251, 247)
SYS16 = (4001, 4331)


def config1(seed: int = DEFAULT_SEED):
    """BASELINE config 1: 56x56x64->64, 3x3 pad 1, F(8,3), RNS(251,241,239)."""
    case = LayerCase("cfg1", 1, 56, 56, 64, 64, 3, 1, 8, SYS8, declared_bound=9 * 64 * 32 * 32)
    rng = make_rng(seed, "cfg1")
    w = uniform_int8(rng, (3, 3, 64, 64), -32, 31)
    x = uniform_int8(rng, (1, 56, 56, 64), -32, 31)
    return case, w, x


def config3(seed: int = DEFAULT_SEED):
    """BASELINE config 3: B=8, 56x56x128->128, 5x5 pad 2, F(8,5), RNS(251,241,239)."""
    case = LayerCase("cfg3", 8, 56, 56, 128, 128, 5, 2, 8, SYS8, declared_bound=25 * 128 * 16 * 16)
    rng = make_rng(seed, "cfg3")
    w = uniform_int8(rng, (5, 5, 128, 128), -16, 15)
    x = uniform_int8(rng, (8, 56, 56, 128), -16, 15)
    return case, w, x


def config5_operands(seed: int = DEFAULT_SEED):
    rng = make_rng(seed, "cfg5")
    w = gaussian_int8(rng, (3, 3, 256, 256))
    x = uniform_int8(rng, (32, 28, 28, 256), 0, 127)
    return w, x


def config5_cases(seed: int = DEFAULT_SEED):
    """BASELINE config 5 sweep: tiles N = 8..16 (M = 6..14) over 2x16-bit and
    3x8-bit RNS wherever the moduli are compatible with the tile
    (253 = 11*23 fails from N = 13 on, 247 = 13*19 from N = 15)."""
    w, _ = config5_operands(seed)
    bound = weight_bound(w, 127)
    cases = []
    for m in (6, 8, 10, 12, 14):
        systems = [SYS16, SYS8] + ([SYS8B] if m + 2 <= 12 else [])
        for mods in systems:
            cases.append(LayerCase(f"cfg5-F{m}-{'x'.join(map(str, mods))}", 32, 28, 28, 256, 256, 3, 1, m, mods,
                                   declared_bound=bound))
    return cases


# ---------------------------------------------------------------------------
# VGG16 (configs 2 and 4): the real 13-layer 3x3 stack on 224x224x3.

VGG16_LAYERS = [
    # name, input side, C, K, pool after
    ("conv1_1", 224, 3, 64, False),
    ("conv1_2", 224, 64, 64, True),
    ("conv2_1", 112, 64, 128, False),
    ("conv2_2", 112, 128, 128, True),
    ("conv3_1", 56, 128, 256, False),
    ("conv3_2", 56, 256, 256, False),
    ("conv3_3", 56, 256, 256, True),
    ("conv4_1", 28, 256, 512, False),
    ("conv4_2", 28, 512, 512, False),
    ("conv4_3", 28, 512, 512, True),
    ("conv5_1", 14, 512, 512, False),
    ("conv5_2", 14, 512, 512, False),
    ("conv5_3", 14, 512, 512, True),
]

# Requantisation shifts between layers: relu, >> s, clip to [0, 127].
# Calibrated once (tools/calibrate_vgg.py) on the seed-2020 weights and image
# so the int8 activations use their range; frozen here so every run, CPU or
# GPU, applies the same glue.
VGG16_SHIFTS = (8, 9, 8, 9, 10, 9, 9, 10, 10, 9, 11, 9, 10)


@dataclass(frozen=True)
class VGGConfig:
    batch: int = 1
    tile_m: int = 14
    moduli: tuple = SYS16
    seed: int = DEFAULT_SEED
    shifts: tuple = VGG16_SHIFTS
    layers: tuple = field(default_factory=lambda: tuple(VGG16_LAYERS))

    def layer_cases(self, bounds=None) -> list[LayerCase]:
        out = []
        for i, (name, side, c, k, _) in enumerate(self.layers):
            out.append(LayerCase(name, self.batch, side, side, c, k, 3, 1, self.tile_m, self.moduli,
                                 declared_bound=None if bounds is None else bounds[i]))
        return out

    def direct_ops(self) -> int:
        return sum(c.direct_ops() for c in self.layer_cases())


def vgg16_weights(seed: int = DEFAULT_SEED) -> list[np.ndarray]:
    """(3,3,C,K) int8 per layer, round(N(0, 20^2)) clipped."""
    # make_rng folds a string label to its first 8 bytes (the reference's
    # rw/cli.py:82-94 convention), so the per-layer / per-image index goes in
    # as its own entropy word: every layer and every image gets its own stream
    return [gaussian_int8(make_rng(seed, "vgg16w", i), (3, 3, c, k)) for i, (_, _, c, k, _) in enumerate(VGG16_LAYERS)]


def vgg16_images(batch: int, seed: int = DEFAULT_SEED, start: int = 0) -> np.ndarray:
    """(batch, 224, 224, 3) int8 images uniform in [0, 127]; image i is drawn
    from its own stream so any shard [start, start+batch) is reproducible."""
    out = np.empty((batch, 224, 224, 3), dtype=np.int8)
    for i in range(batch):
        out[i] = uniform_int8(make_rng(seed, "vgg16img", start + i), (224, 224, 3), 0, 127)
    return out


def vgg16_bounds(weights, moduli=SYS16) -> list[int]:
    """Per-layer declared bound: the sound weight-derived bound (inputs are in
    [0,127]) when it fits the system, else the system's signed bound, in which
    case exactness rests on the mandatory direct-conv comparison (SURVEY.md
    8(d), config 2)."""
    import math

    sb = (math.prod(moduli) - 1) // 2
    return [min(weight_bound(w, 127), sb) for w in weights]


# ---------------------------------------------------------------------------
# The reference's verification sweep (rw/cli.py:259-314): 12 (tile, filter)
# shapes x 3 moduli sets x 7 seeded geometries, minus combinations whose
# transform denominators share a factor with a modulus.

VERIFY_SYSTEMS = ((253, 251, 247), (251, 241, 239), (4001, 4331))
VERIFY_SHAPES = ((2, 3), (4, 3), (8, 3), (10, 3), (12, 3), (14, 3),
                 (2, 5), (4, 5), (8, 5), (10, 5), (12, 5), (14, 5))


def verify_cases(seed: int = DEFAULT_SEED) -> list[dict]:
    from .transforms import cached_transforms, check_modulus_compatibility

    geo = make_rng(seed, "geometry")
    out = []
    for tile_m, r in VERIFY_SHAPES:
        ts = cached_transforms(tile_m, r)
        for mods in VERIFY_SYSTEMS:
            if not all(check_modulus_compatibility(ts, m) for m in mods):
                continue
            for g in range(7):
                # draw order matters: h, w, c, k, padding, batch
                h, w = int(geo.integers(r, 33)), int(geo.integers(r, 33))
                c, k = int(geo.integers(1, 17)), int(geo.integers(1, 9))
                pad, batch = int(geo.integers(0, 3)), int(geo.integers(1, 3))
                out.append(dict(tile_m=tile_m, r=r, moduli=mods, h=h, w=w, c=c, k=k, pad=pad, batch=batch,
                                entropy=(seed, tile_m, r, *mods, g)))
    return out


def verify_operands(case: dict):
    """Weights then activations in [-127, 127] from the case's own stream
    (rw/cli.py:317-322, 97-99)."""
    rng = make_rng(*case["entropy"])
    w = rng.integers(-127, 128, size=(case["r"], case["r"], case["c"], case["k"]), dtype=np.int8)
    x = rng.integers(-127, 128, size=(case["batch"], case["h"], case["w"], case["c"]), dtype=np.int8)
    return w, x
