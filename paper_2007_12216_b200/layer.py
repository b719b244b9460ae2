"""The reference's layer entry point, backed by sm_100a kernels.

Mirrors rw/layer.py's public surface for the hot path -- ``LayerSpec``,
``range_check``/``RangeReport``, ``StageTimings``,
``precompute_filter_transforms`` and ``winograd_layer_conv`` /
``layer_conv`` -- with the same argument meaning, the same pre-flight checks
in the same order and the same exception classes (rw/layer.py:31-412).  The
arithmetic happens in librnsw.so (include/rnsw.h); this module only checks
arguments, builds plans and moves buffers.

Operands may be numpy arrays (the reference's types: results come back as
numpy int32) or torch tensors (results stay on the GPU).  The north-star
front door ``conv2d_rns`` takes NCHW activations and OIHW weights and runs the
same kernels with NCHW addressing; no permutation copies are made.
"""

from __future__ import annotations

import threading
from collections.abc import Mapping
from dataclasses import dataclass
from fractions import Fraction
from math import ceil
from typing import Sequence

import numpy as np

from . import _native, transforms
from .errors import DynamicRangeExceeded, ShapeMismatch, UnsupportedStride
from .residue import RnsSystem

INT8_PEAK = 127


def _torch():
    import torch

    return torch


# ---------------------------------------------------------------------------
# geometry and pre-flight checks (rw/layer.py:31-78, 177-208)


@dataclass(frozen=True)
class LayerSpec:
    """One convolution layer: square filter r x r, NHWC activations."""

    h: int
    w: int
    c: int
    k: int
    r: int
    batch: int = 1
    padding: int = 0
    stride: int = 1
    tile_m: int | None = None

    def __post_init__(self):
        for name in ("h", "w", "c", "k", "r", "batch", "stride"):
            v = getattr(self, name)
            if isinstance(v, bool) or not isinstance(v, int) or v < 1:
                raise ValueError(f"{name} must be a positive integer, got {v!r}")
        if isinstance(self.padding, bool) or not isinstance(self.padding, int) or self.padding < 0:
            raise ValueError(f"padding must be a non-negative integer, got {self.padding!r}")
        if self.h + 2 * self.padding < self.r or self.w + 2 * self.padding < self.r:
            raise ValueError("padded input smaller than the filter")
        if self.tile_m is not None and (isinstance(self.tile_m, bool) or not isinstance(self.tile_m, int)
                                        or self.tile_m < 1):
            raise ValueError(f"tile_m must be a positive integer, got {self.tile_m!r}")

    @property
    def out_h(self) -> int:
        return (self.h + 2 * self.padding - self.r) // self.stride + 1

    @property
    def out_w(self) -> int:
        return (self.w + 2 * self.padding - self.r) // self.stride + 1

    def weight_shape(self) -> tuple[int, int, int, int]:
        return (self.r, self.r, self.c, self.k)

    def input_shape(self) -> tuple[int, int, int, int]:
        return (self.batch, self.h, self.w, self.c)

    def tiles(self, tile_m: int | None = None) -> int:
        m = self.tile_m if tile_m is None else tile_m
        return self.batch * ceil(self.out_h / m) * ceil(self.out_w / m)


@dataclass(frozen=True)
class RangeReport:
    static_bound: int
    declared_bound: int | None
    bound: int
    signed_bound: int

    @property
    def fits(self) -> bool:
        return self.bound <= self.signed_bound


def range_check(spec: LayerSpec, system: RnsSystem, declared_bound: int | None = None) -> RangeReport:
    """Static worst case r*r*c*127^2 unless the caller declares a bound
    (rw/layer.py:191-208).  A false declaration wraps the output modulo the
    dynamic range, exactly like the reference (SURVEY.md finding 3)."""
    static = spec.r * spec.r * spec.c * INT8_PEAK * INT8_PEAK
    bound = static if declared_bound is None else declared_bound
    return RangeReport(static_bound=static, declared_bound=declared_bound, bound=bound,
                       signed_bound=system.signed_bound)


@dataclass
class StageTimings:
    """Seconds per stage.  Device stages are timed with CUDA events on the
    launching stream (the reference uses perf_counter, rw/layer.py:211-232)."""

    tiling: float = 0.0
    filter_transform: float = 0.0
    input_transform: float = 0.0
    gemm: float = 0.0
    backward_transform: float = 0.0
    mrc: float = 0.0
    scatter: float = 0.0

    def total(self) -> float:
        return (self.tiling + self.filter_transform + self.input_transform + self.gemm
                + self.backward_transform + self.mrc + self.scatter)


@dataclass(frozen=True)
class OperationCounts:
    direct_mults: int
    winograd_mults: int
    tiles: int
    reduction_ratio: Fraction


def count_operations(spec: LayerSpec, system: RnsSystem, tile_m: int | None = None) -> OperationCounts:
    """GEMM multiplication counts, direct vs tiled (rw/layer.py:425-450)."""
    tile_m = spec.tile_m if tile_m is None else tile_m
    if tile_m is None:
        raise ValueError("tile_m must be given (argument or spec.tile_m)")
    n = tile_m + spec.r - 1
    tiles = spec.tiles(tile_m)
    direct = spec.batch * spec.out_h * spec.out_w * spec.k * spec.c * spec.r * spec.r
    wino = tiles * n * n * spec.c * spec.k * len(system.moduli)
    return OperationCounts(direct, wino, tiles, Fraction(direct, wino))


@dataclass(frozen=True)
class TilePlacement:
    """Where one patch's outputs land in the layer output plane (rw/layer.py:106-115)."""

    row: int
    col: int
    out_h0: int
    out_h1: int
    out_w0: int
    out_w1: int


def tile_decompose(x, tile_m: int, r: int, padding: int):
    """Overlapping n x n patches (n = tile_m + r - 1) of the zero canvas at
    stride tile_m, and each patch's crop rectangle (rw/layer.py:118-158).

    The layer path never materialises the patches (the input-transform kernel
    addresses the canvas directly); this public counterpart gathers them on
    the GPU (rnsw_tile_decompose).  numpy in -> numpy patches; torch in ->
    device tensor.  Returns (patches (B, th, tw, n, n, C) int8, placements)."""
    torch = _torch()
    if len(x.shape) != 4:
        raise ShapeMismatch(f"x must be (b, h, w, c), got {tuple(x.shape)}")
    if not _is_int8(x):
        raise ShapeMismatch(f"x must be int8, got {x.dtype}")
    b, h, w, c = (int(v) for v in x.shape)
    n = tile_m + r - 1
    out_h, out_w = h + 2 * padding - r + 1, w + 2 * padding - r + 1
    if out_h < 1 or out_w < 1:
        raise ShapeMismatch("padded input smaller than the filter")
    th, tw = ceil(out_h / tile_m), ceil(out_w / tile_m)
    host_result = isinstance(x, np.ndarray)
    xd = to_device(x)
    patches = torch.empty((b, th, tw, n, n, c), dtype=torch.int8, device=xd.device)
    l = _native.lib()
    _native.check(l.rnsw_tile_decompose(_native.c_void_p(xd.data_ptr()), b, h, w, c, tile_m, r, padding,
                                        _native.c_void_p(patches.data_ptr()), patches.numel(), _stream_ptr()))
    placements = [TilePlacement(row=ti, col=tj, out_h0=ti * tile_m, out_h1=min(ti * tile_m + tile_m, out_h),
                                out_w0=tj * tile_m, out_w1=min(tj * tile_m + tile_m, out_w))
                  for ti in range(th) for tj in range(tw)]
    return (patches.cpu().numpy() if host_result else patches), placements


# ---------------------------------------------------------------------------
# plans and operand handling

_plans: dict = {}
_plans_lock = threading.Lock()


def plan_for(ts: transforms.ExactTransformSet, system: RnsSystem) -> _native.Plan:
    """Native plan for (transform set, system) on the current CUDA device."""
    torch = _torch()
    mts = _modular_sets(ts, system)  # NotCoprime surfaces here, before any device work
    dev = torch.cuda.current_device()
    key = (ts.m, ts.r, ts.points, system.moduli, dev)
    plan = _plans.get(key)
    if plan is None:
        plan = plan_from_modular(mts, system)
        with _plans_lock:
            _plans.setdefault(key, plan)
            plan = _plans[key]
    return plan


_mts_cache: dict = {}


def _modular_sets(ts: transforms.ExactTransformSet, system: RnsSystem):
    key = (ts.m, ts.r, ts.points, system.moduli)
    mts = _mts_cache.get(key)
    if mts is None:
        mts = transforms.reduce_for_system(ts, system)
        _mts_cache[key] = mts
    return mts


def plan_from_modular(mts: Sequence[transforms.ModularTransformSet], system: RnsSystem) -> _native.Plan:
    at = np.stack([mt.at.astype(np.int16) for mt in mts])
    g = np.stack([mt.g.astype(np.int16) for mt in mts])
    bt = np.stack([mt.bt.astype(np.int16) for mt in mts])
    return _native.Plan(mts[0].m, mts[0].r, system.moduli, at, g, bt, system.mrc_table())


def _shape(a) -> tuple:
    return tuple(a.shape)


def _is_int8(a) -> bool:
    if isinstance(a, np.ndarray):
        return a.dtype == np.int8
    torch = _torch()
    return isinstance(a, torch.Tensor) and a.dtype == torch.int8


def _check_operands(spec: LayerSpec, weights, x, weight_shape=None, input_shape=None) -> None:
    ws = spec.weight_shape() if weight_shape is None else weight_shape
    xs = spec.input_shape() if input_shape is None else input_shape
    if _shape(weights) != ws:
        raise ShapeMismatch(f"weights {_shape(weights)} do not match {ws}")
    if _shape(x) != xs:
        raise ShapeMismatch(f"input {_shape(x)} does not match {xs}")
    if not (_is_int8(weights) and _is_int8(x)):
        raise ShapeMismatch(f"operands must be int8, got {weights.dtype} and {x.dtype}")


def to_device(a, non_blocking: bool = False):
    """numpy / CPU tensor -> contiguous CUDA tensor on the current device."""
    torch = _torch()
    if isinstance(a, np.ndarray):
        a = torch.from_numpy(np.ascontiguousarray(a))
    if not a.is_cuda:
        a = a.to(f"cuda:{torch.cuda.current_device()}", non_blocking=non_blocking)
    return a.contiguous()


def _stream_ptr():
    torch = _torch()
    return _native.c_void_p(torch.cuda.current_stream().cuda_stream)


class FilterBank(Mapping):
    """Transformed filters resident on the GPU, in the tensor-core layout
    [plane][pos][K][Cp] (``precompute_filter_transforms`` output).

    Indexing by modulus returns that residue's filters in the reference layout
    (N, N, C, K) as a host numpy array, so code written against the reference
    dict keeps working (rw/layer.py:161-174); the layer path uses ``data``
    directly.
    """

    def __init__(self, plan: _native.Plan, data, c: int, k: int):
        self.plan, self.data, self.c, self.k = plan, data, int(c), int(k)
        self.moduli = plan.moduli
        self.n = plan.n

    def __getitem__(self, m):
        """The reference dict's value: int8 residues for m < 256, int16
        otherwise (dtype_for_modulus, rw/gemm.py:25-27; rw/transforms.py:303-313)."""
        if m not in self.moduli:
            raise KeyError(m)
        u = self.device_view(m).cpu().numpy()
        return u.astype(np.int8) if m < 256 else u

    def __iter__(self):
        return iter(self.moduli)

    def __len__(self) -> int:
        return len(self.moduli)

    @staticmethod
    def bank_planes(m) -> int:
        """Planes per residue in the bank: u itself for m < 256; otherwise the
        limbs of u and of 256*u mod m (consumed by the 2-accumulator GEMM)."""
        return 1 if m < 256 else 4

    def planes_of(self, m) -> tuple[int, int]:
        base = 0
        for mod in self.moduli:
            pl = self.bank_planes(mod)
            if mod == m:
                return base, pl
            base += pl
        raise KeyError(m)

    def device_view(self, m):
        """(N, N, C, K) int16 symmetric residues of modulus m, on the GPU."""
        torch = _torch()
        n, c, k = self.n, self.c, self.k
        total = sum(self.bank_planes(mod) for mod in self.moduli)
        cp = self.data.numel() // (total * n * n * k)
        u = self.data.view(torch.int8).view(total, n * n, k, cp)[..., :c]
        base, pl = self.planes_of(m)
        v = u[base].to(torch.int16)
        if pl > 1:
            v = u[base + 1].to(torch.int16) * 256 + v
        return v.permute(0, 2, 1).reshape(n, n, c, k).contiguous()


def _filters_on_device(plan: _native.Plan, weights_dev, c: int, k: int, layout: int) -> FilterBank:
    torch = _torch()
    l = _native.lib()
    nbytes = l.rnsw_filter_bytes(plan.handle, c, k)
    u = torch.empty(nbytes, dtype=torch.uint8, device=weights_dev.device)
    _native.check(l.rnsw_filter_transform(plan.handle, _native.c_void_p(weights_dev.data_ptr()), c, k, layout,
                                          _native.c_void_p(u.data_ptr()), nbytes, _stream_ptr()))
    return FilterBank(plan, u, c, k)


def precompute_filter_transforms(weights, mts: Sequence[transforms.ModularTransformSet]) -> FilterBank:
    """U = G g G^T mod m for every modulus, computed once on the GPU
    (rw/layer.py:161-174).  ``weights`` is (R, R, C, K) int8."""
    if len(weights.shape) != 4 or weights.shape[0] != weights.shape[1]:
        raise ShapeMismatch(f"weights must be (r, r, c, k), got {tuple(weights.shape)}")
    if not _is_int8(weights):
        raise ShapeMismatch(f"weights must be int8, got {weights.dtype}")
    system = RnsSystem([mt.modulus for mt in mts])
    plan = plan_from_modular(mts, system)
    r, _, c, k = (int(s) for s in weights.shape)
    if r != plan.r:
        raise ShapeMismatch(f"filters are {r}x{r}, transform sets expect r={plan.r}")
    return _filters_on_device(plan, to_device(weights), c, k, _native.LAYOUT_NHWC)


def _bank_for(plan: _native.Plan, filters, spec_c: int, spec_k: int, n: int):
    """Validate ``filters`` like rw/layer.py:350-358 and return the device bank."""
    torch = _torch()
    if isinstance(filters, FilterBank) and filters.plan.moduli == plan.moduli and filters.n == n \
            and filters.plan.tile_m == plan.tile_m and filters.plan.r == plan.r \
            and (filters.plan is plan or filters.plan.key == plan.key):
        if filters.c != spec_c or filters.k != spec_k:
            raise ShapeMismatch(f"precomputed filters are for c={filters.c}, k={filters.k}; "
                                f"layer needs ({n}, {n}, {spec_c}, {spec_k})")
        return filters.data
    l = _native.lib()
    nbytes = l.rnsw_filter_bytes(plan.handle, spec_c, spec_k)
    u = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{torch.cuda.current_device()}")
    for i, m in enumerate(plan.moduli):
        f = filters.get(m) if isinstance(filters, Mapping) else None
        if f is None or tuple(f.shape) != (n, n, spec_c, spec_k):
            raise ShapeMismatch(f"precomputed filters for modulus {m} missing or not shaped "
                                f"({n}, {n}, {spec_c}, {spec_k})")
        src = f.to(torch.int16) if isinstance(f, torch.Tensor) else torch.from_numpy(np.asarray(f, dtype=np.int16))
        src = to_device(src)
        _native.check(l.rnsw_filter_import(plan.handle, i, _native.c_void_p(src.data_ptr()), spec_c, spec_k,
                                           _native.c_void_p(u.data_ptr()), nbytes, _stream_ptr()))
    return u


# ---------------------------------------------------------------------------
# the layer


_ws_local = threading.local()


def _workspace(nbytes: int, device):
    """Per-thread, per-(device, stream) workspace that grows on demand, so
    repeated layer calls do not allocate (calls on one stream are ordered, so
    reusing the buffer is safe; other threads / streams get their own)."""
    torch = _torch()
    cache = getattr(_ws_local, "bufs", None)
    if cache is None:
        cache = _ws_local.bufs = {}
    key = (str(device), torch.cuda.current_stream(device).cuda_stream)
    buf = cache.get(key)
    if buf is None or buf.numel() < nbytes:
        cache.pop(key, None)
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        cache[key] = buf
    return buf


def _run_layer(plan, x_dev, b, h, w, c, k, pad, layout, bank, timings: StageTimings | None):
    """Launch the device stages (rnsw_conv_forward); returns the int32 output
    tensor.  With ``timings`` the same kernel chain runs through
    rnsw_conv_forward_timed, which records CUDA events between the stages."""
    torch = _torch()
    l = _native.lib()
    ho, wo = h + 2 * pad - plan.r + 1, w + 2 * pad - plan.r + 1
    shape = (b, ho, wo, k) if layout == _native.LAYOUT_NHWC else (b, k, ho, wo)
    y = torch.empty(shape, dtype=torch.int32, device=x_dev.device)
    ws_bytes = l.rnsw_workspace_bytes(plan.handle, b, h, w, c, k, pad)
    if ws_bytes == 0:
        raise ShapeMismatch("layer geometry rejected by the native plan")
    ws = _workspace(ws_bytes, x_dev.device)
    s = _stream_ptr()
    vp = _native.c_void_p
    if timings is None:
        _native.check(l.rnsw_conv_forward(plan.handle, vp(x_dev.data_ptr()), b, h, w, c, k, pad, layout,
                                          vp(bank.data_ptr()), vp(y.data_ptr()), vp(ws.data_ptr()), ws.numel(), s))
        return y
    ms = (_native.ctypes.c_float * 3)()
    _native.check(l.rnsw_conv_forward_timed(plan.handle, vp(x_dev.data_ptr()), b, h, w, c, k, pad, layout,
                                            vp(bank.data_ptr()), vp(y.data_ptr()), vp(ws.data_ptr()), ws.numel(), s,
                                            ms))
    timings.input_transform += ms[0] / 1e3
    timings.gemm += ms[1] / 1e3
    # backward transform, MRC and scatter are one fused kernel on the device
    timings.backward_transform += ms[2] / 1e3
    return y


def _to_host(y):
    """Device int32 result -> numpy through a pinned staging buffer."""
    torch = _torch()
    host = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
    host.copy_(y, non_blocking=True)
    torch.cuda.current_stream(y.device).synchronize()
    return host.numpy()


def winograd_layer_conv(spec: LayerSpec, weights, x, system: RnsSystem, declared_bound: int | None = None,
                        transform_set: transforms.ExactTransformSet | None = None, filters=None,
                        timings: StageTimings | None = None):
    """Exact integer convolution through the tiled RNS-Winograd path on the GPU.

    Same contract as rw/layer.py:301-389: ``weights`` (R,R,C,K) and ``x``
    (B,H,W,C) int8, result (B,Ho,Wo,K) int32 -- numpy in, numpy out; torch in,
    torch (on the GPU) out.  Raises ShapeMismatch, UnsupportedStride,
    ValueError (no tile_m), DynamicRangeExceeded, NotCoprime in that order.
    """
    _check_operands(spec, weights, x)
    if spec.stride != 1:
        raise UnsupportedStride(f"fast path needs stride 1, got {spec.stride}")
    if spec.tile_m is None:
        raise ValueError("spec.tile_m must be set for the fast path")
    report = range_check(spec, system, declared_bound)
    if not report.fits:
        raise DynamicRangeExceeded(f"worst case {report.bound} exceeds signed bound {report.signed_bound}")
    if transform_set is None:
        transform_set = transforms.cached_transforms(spec.tile_m, spec.r)
    if transform_set.m != spec.tile_m or transform_set.r != spec.r:
        raise ShapeMismatch(f"transform set is for ({transform_set.m}, {transform_set.r}), "
                            f"layer needs ({spec.tile_m}, {spec.r})")
    plan = plan_for(transform_set, system)
    host_result = isinstance(x, np.ndarray)
    x_dev = to_device(x)
    n = spec.tile_m + spec.r - 1
    if filters is None:
        bank = _filters_on_device(plan, to_device(weights), spec.c, spec.k, _native.LAYOUT_NHWC).data
    else:
        bank = _bank_for(plan, filters, spec.c, spec.k, n)
    y = _run_layer(plan, x_dev, spec.batch, spec.h, spec.w, spec.c, spec.k, spec.padding, _native.LAYOUT_NHWC,
                   bank, timings)
    return _to_host(y) if host_result else y


def _c16(c: int) -> int:
    return (c + 15) // 16 * 16


class DirectWeights:
    """Weights packed once for the direct tcgen05 convolution ([K][R*R*Cp]).
    Channel counts that are not a multiple of 16 are zero-padded to one (the
    activations get the same zero channels in ``direct_conv``), so every C
    runs on the device."""

    def __init__(self, weights, layout: int = _native.LAYOUT_NHWC):
        torch = _torch()
        wd = to_device(weights)
        if layout == _native.LAYOUT_NHWC:
            r, _, c, k = (int(v) for v in wd.shape)
            if c % 16:
                wp = torch.zeros((r, r, _c16(c), k), dtype=torch.int8, device=wd.device)
                wp[:, :, :c, :] = wd
                wd = wp
        else:
            k, c, r, _ = (int(v) for v in wd.shape)
            if c % 16:
                wp = torch.zeros((k, _c16(c), r, r), dtype=torch.int8, device=wd.device)
                wp[:, :c] = wd
                wd = wp
        cp = _c16(c)
        l = _native.lib()
        nbytes = l.rnsw_direct_weight_bytes(r, cp, k)
        self.data = torch.empty(nbytes, dtype=torch.int8, device=wd.device)
        _native.check(l.rnsw_direct_pack_weights(_native.c_void_p(wd.data_ptr()), r, cp, k, layout,
                                                 _native.c_void_p(self.data.data_ptr()), nbytes, _stream_ptr()))
        self.r, self.c, self.k = r, c, k


def direct_conv(spec: LayerSpec, weights, x, packed: DirectWeights | None = None):
    """Exact int32 convolution on the tensor cores: the device counterpart of
    the reference's oracle direct_conv (rw/layer.py:93-103), any stride and
    any C (channels zero-padded to a multiple of 16 on the device for the TMA
    row alignment).  Implicit GEMM on tcgen05 kind::i8 with TMA im2col boxes."""
    torch = _torch()
    _check_operands(spec, weights, x)
    host_result = isinstance(x, np.ndarray)
    xd = to_device(x)
    if packed is None:
        packed = DirectWeights(weights)
    c = spec.c
    if c % 16:
        xp = torch.zeros((spec.batch, spec.h, spec.w, _c16(c)), dtype=torch.int8, device=xd.device)
        xp[..., :c] = xd
        xd, c = xp, _c16(c)
    y = torch.empty((spec.batch, spec.out_h, spec.out_w, spec.k), dtype=torch.int32, device=xd.device)
    l = _native.lib()
    _native.check(l.rnsw_direct_conv(_native.c_void_p(xd.data_ptr()), spec.batch, spec.h, spec.w, c,
                                     _native.c_void_p(packed.data.data_ptr()), spec.k, spec.r, spec.padding,
                                     spec.stride, _native.c_void_p(y.data_ptr()), _stream_ptr()))
    return _to_host(y) if host_result else y


def layer_conv(spec: LayerSpec, weights, x, system: RnsSystem, declared_bound: int | None = None, filters=None,
               timings: StageTimings | None = None):
    """rw/layer.py:392-412: stride != 1 goes to the direct convolution --
    here the tcgen05 implicit-GEMM kernel, not a CPU fallback."""
    if spec.stride != 1:
        return direct_conv(spec, weights, x)
    return winograd_layer_conv(spec, weights, x, system, declared_bound=declared_bound, filters=filters,
                               timings=timings)


def conv2d_rns(x_nchw, w_oihw, moduli, tile_m: int, padding: int = 0, declared_bound: int | None = None,
               filters=None):
    """North-star front door: NCHW int8 activations, OIHW int8 weights, a
    moduli set and a tile size in; exact NCHW int32 out.

    Identical semantics to ``winograd_layer_conv`` on the permuted operands
    (x_nhwc = x.transpose(0,2,3,1), w_rrck = w.transpose(2,3,1,0)); the
    kernels address NCHW/OIHW directly.  ``filters`` may be a FilterBank from
    ``precompute_filters_oihw``.
    """
    system = moduli if isinstance(moduli, RnsSystem) else RnsSystem(moduli)
    if len(x_nchw.shape) != 4 or len(w_oihw.shape) != 4:
        raise ShapeMismatch("conv2d_rns takes NCHW activations and OIHW weights")
    b, c, h, w = (int(s) for s in x_nchw.shape)
    k, c2, r, r2 = (int(s) for s in w_oihw.shape)
    if r != r2:
        raise ShapeMismatch(f"filters must be square, got {r}x{r2}")
    spec = LayerSpec(h=h, w=w, c=c, k=k, r=r, batch=b, padding=padding, tile_m=tile_m)
    _check_operands(spec, w_oihw, x_nchw, weight_shape=(k, c, r, r), input_shape=(b, c, h, w))
    report = range_check(spec, system, declared_bound)
    if not report.fits:
        raise DynamicRangeExceeded(f"worst case {report.bound} exceeds signed bound {report.signed_bound}")
    plan = plan_for(transforms.cached_transforms(tile_m, r), system)
    host_result = isinstance(x_nchw, np.ndarray)
    x_dev = to_device(x_nchw)
    if filters is None:
        bank = _filters_on_device(plan, to_device(w_oihw), c, k, _native.LAYOUT_NCHW).data
    else:
        bank = _bank_for(plan, filters, c, k, plan.n)
    y = _run_layer(plan, x_dev, b, h, w, c, k, padding, _native.LAYOUT_NCHW, bank, None)
    return _to_host(y) if host_result else y


def precompute_filters_oihw(w_oihw, moduli, tile_m: int) -> FilterBank:
    """FilterBank from OIHW weights (the conv2d_rns counterpart of
    precompute_filter_transforms)."""
    system = moduli if isinstance(moduli, RnsSystem) else RnsSystem(moduli)
    k, c, r, _ = (int(s) for s in w_oihw.shape)
    if not _is_int8(w_oihw):
        raise ShapeMismatch(f"weights must be int8, got {w_oihw.dtype}")
    plan = plan_for(transforms.cached_transforms(tile_m, r), system)
    return _filters_on_device(plan, to_device(w_oihw), c, k, _native.LAYOUT_NCHW)
