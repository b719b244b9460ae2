"""VGG16 conv stack on the RNS-Winograd device path (BASELINE configs 2 and 4).

Thirteen 3x3/pad-1 layers, each an exact int32 RNS-Winograd convolution
(F(14x14,3x3) over RNS(4001,4331) by default) followed by the device glue
relu -> >> shift -> clip [0,127] (-> 2x2 max-pool after each block).  The
glue is defined by BASELINE.json, not by the reference package.
Filters are transformed once at construction (the reference bench also
excludes the filter transform from timing, rw/cli.py:459-472).

Everything runs on one CUDA stream; buffers are allocated once per batch size
so a forward pass issues only kernel launches (52 for the 13 layers).
"""

from __future__ import annotations

import math

from . import _native, workloads
from .layer import _filters_on_device, _stream_ptr, plan_for, range_check, LayerSpec
from .errors import DynamicRangeExceeded
from .residue import RnsSystem
from .transforms import cached_transforms


def _torch():
    import torch

    return torch


class VGG16Rns:
    def __init__(self, cfg: workloads.VGGConfig | None = None, weights=None):
        torch = _torch()
        self.cfg = cfg or workloads.VGGConfig()
        self.system = RnsSystem(self.cfg.moduli)
        self.plan = plan_for(cached_transforms(self.cfg.tile_m, 3), self.system)
        self.weights = weights if weights is not None else workloads.vgg16_weights(self.cfg.seed)
        self.bounds = workloads.vgg16_bounds(self.weights, self.cfg.moduli)
        self.banks = []
        for (name, side, c, k, _), w, bound in zip(self.cfg.layers, self.weights, self.bounds):
            spec = LayerSpec(h=side, w=side, c=c, k=k, r=3, padding=1, tile_m=self.cfg.tile_m)
            rep = range_check(spec, self.system, bound)
            if not rep.fits:
                raise DynamicRangeExceeded(f"{name}: bound {rep.bound} exceeds {rep.signed_bound}")
            wd = torch.from_numpy(w).cuda()
            self.banks.append(_filters_on_device(self.plan, wd, c, k, _native.LAYOUT_NHWC))
        torch.cuda.synchronize()
        self._buffers = {}

    def _alloc(self, batch: int):
        torch = _torch()
        if batch in self._buffers:
            return self._buffers[batch]
        l = _native.lib()
        dev = f"cuda:{torch.cuda.current_device()}"
        ws = max(l.rnsw_workspace_bytes(self.plan.handle, batch, side, side, c, k, 1)
                 for _, side, c, k, _ in self.cfg.layers)
        ymax = max(batch * side * side * k for _, side, c, k, _ in self.cfg.layers)
        amax = max(batch * side * side * c for _, side, c, k, _ in self.cfg.layers)
        bufs = {
            "ws": torch.empty(ws, dtype=torch.uint8, device=dev),
            "y": torch.empty(ymax, dtype=torch.int32, device=dev),
            "act": [torch.empty(amax, dtype=torch.int8, device=dev) for _ in range(2)],
            "out": torch.empty((batch, 7, 7, 512), dtype=torch.int8, device=dev),
        }
        self._buffers[batch] = bufs
        return bufs

    def launches_per_forward(self) -> int:
        return 4 * len(self.cfg.layers)  # input transform, GEMM, output transform, glue

    def launches_fused(self) -> int:
        """Kernels per forward_fused: input transform, product (GEMM or the
        C <= 4 CUDA-core product), output transform with the glue."""
        return 3 * len(self.cfg.layers)

    def layer_work(self, batch: int, fused: bool = False) -> list[dict]:
        """Algorithmic work per layer and kernel ("Roofline"):
        bytes for the memory-bound stages, int8 tensor ops for the GEMM."""
        out = []
        n = self.plan.n
        npos = n * n
        planes = sum(1 if m < 256 else 2 for m in self.cfg.moduli)
        mma_per_product = sum(1 if m < 256 else 4 for m in self.cfg.moduli)
        for name, side, c, k, pool in self.cfg.layers:
            tiles = batch * math.ceil(side / self.cfg.tile_m) ** 2
            oside = side // 2 if pool else side
            out.append({
                "name": name,
                "input_transform_bytes": batch * side * side * c + planes * npos * tiles * c,
                "gemm_ops": 2 * tiles * npos * c * k * mma_per_product,
                # V in, the filter residues once (one byte per 8-bit modulus, two per
                # 16-bit one: the tile-row GEMM also streams the two derived 256 u mod m
                # planes, the small-P GEMM does not), the Winograd-domain product out
                "gemm_bytes": planes * npos * tiles * c + planes * npos * k * c
                + len(self.cfg.moduli) * npos * tiles * k * 2,
                "output_transform_bytes": len(self.cfg.moduli) * npos * tiles * k * 2 + (
                    batch * oside * oside * k if fused else batch * side * side * k * 4),
                "glue_bytes": batch * side * side * k * 4 + batch * oside * oside * k,
                # C <= 4 layers run the CUDA-core product (csrc/smallc.cu): V16 in, Mw out
                "product_bytes": len(self.cfg.moduli) * npos * tiles * (8 + 2 * k),
                "direct_ops": 2 * batch * side * side * c * k * 9,
            })
        return out

    def _mw8(self) -> bool:
        """Whether the whole-layer path hands the product to the tcgen05
        output transform in the planar Mw8 layout (include/rnsw.h)."""
        return _native.lib().rnsw_mw8_supported(self.plan.handle) == 1

    def forward_staged(self, x, record):
        """forward() with CUDA events between the kernels of every layer
        (``record(kind, layer, start, end)``), the glue kernel separately."""
        torch = _torch()
        l = _native.lib()
        vp = _native.c_void_p
        batch = int(x.shape[0])
        bufs = self._alloc(batch)
        s = _stream_ptr()
        ws = bufs["ws"]
        cur = x.contiguous()
        nl = len(self.cfg.layers)
        for i, ((name, side, c, k, pool), bank) in enumerate(zip(self.cfg.layers, self.banks)):
            y = bufs["y"][: batch * side * side * k].view(batch, side, side, k)
            ev, handles = self._layer_events()
            ev[0].record()
            _native.check(l.rnsw_conv_forward_ev(self.plan.handle, vp(cur.data_ptr()), batch, side, side, c, k, 1,
                                                 _native.LAYOUT_NHWC, vp(bank.data.data_ptr()), vp(y.data_ptr()),
                                                 vp(ws.data_ptr()), ws.numel(), s, handles))
            ev[3].record()
            record("input_transform", i, ev[0], ev[1])
            record("product" if c <= 4 else "gemm", i, ev[1], ev[2])
            record("output_transform", i, ev[2], ev[3])
            oside = side // 2 if pool else side
            nxt = bufs["out"] if i == nl - 1 else \
                bufs["act"][i % 2][: batch * oside * oside * k].view(batch, oside, oside, k)
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            _native.check(l.rnsw_requant_pool(vp(y.data_ptr()), batch, side, side, k, self.cfg.shifts[i],
                                              1 if pool else 0, vp(nxt.data_ptr()), s))
            g1.record()
            record("glue", i, g0, g1)
            cur = nxt
        return cur

    def forward_fused(self, x):
        """Same stack with the glue fused into each layer's output stage
        (rnsw_conv_forward_requant): the int32 outputs are never written.
        Bit-identical to forward() (tests/test_gpu_configs.py)."""
        l = _native.lib()
        vp = _native.c_void_p
        batch = int(x.shape[0])
        bufs = self._alloc(batch)
        s = _stream_ptr()
        ws = bufs["ws"]
        cur = x.contiguous()
        nl = len(self.cfg.layers)
        for i, ((name, side, c, k, pool), bank) in enumerate(zip(self.cfg.layers, self.banks)):
            oside = side // 2 if pool else side
            nxt = bufs["out"] if i == nl - 1 else \
                bufs["act"][i % 2][: batch * oside * oside * k].view(batch, oside, oside, k)
            _native.check(l.rnsw_conv_forward_requant(self.plan.handle, vp(cur.data_ptr()), batch, side, side, c, k,
                                                      1, vp(bank.data.data_ptr()), self.cfg.shifts[i],
                                                      1 if pool else 0, vp(nxt.data_ptr()), vp(ws.data_ptr()),
                                                      ws.numel(), s))
            cur = nxt
        return cur

    def graph(self, x, bind: bool = False):
        """Capture forward_fused(x) for x's shape into a CUDA graph (buffers
        are preallocated per batch size, so replays reuse the same pointers).
        Returns a callable that copies new input into the captured input
        buffer, replays, and returns the captured output tensor.  With
        ``bind`` the graph reads ``x`` itself (no input copy; one graph per
        input buffer)."""
        torch = _torch()
        batch = int(x.shape[0])
        key = ("graph", batch, x.data_ptr() if bind else None)
        if key not in self._buffers:
            if bind:
                static_in = x
            else:
                static_in = torch.empty_like(x)
                static_in.copy_(x)
            # warm up (lazy module loading, attribute setting) outside capture
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                for _ in range(2):
                    self.forward_fused(static_in)
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                static_out = self.forward_fused(static_in)
            self._buffers[key] = (g, static_in, static_out)
        g, static_in, static_out = self._buffers[key]

        def run(new_x=None):
            if new_x is not None and new_x.data_ptr() != static_in.data_ptr():
                static_in.copy_(new_x, non_blocking=True)
            g.replay()
            return static_out

        return run

    def run_stream(self, host_batches, host_outs, post=None) -> None:
        """Serve a sequence of pinned host batches (B, 224, 224, 3) int8 into
        pinned host outputs: each batch's H2D copy and the previous batch's
        D2H copy run on a copy stream while the current batch computes (two
        device input / output buffers, one CUDA graph per input buffer).
        ``post`` maps the (B, 7, 7, 512) device result before it is copied
        out (e.g. the multi-GPU gather); a None output entry skips the D2H.
        Enqueues everything on the current stream and returns; the caller
        synchronizes."""
        torch = _torch()
        n = len(host_batches)
        if n == 0:
            return
        if len(host_outs) != n:
            raise ValueError("one output buffer per batch")
        shape = tuple(host_batches[0].shape)
        comp = torch.cuda.current_stream()
        key = ("stream", shape)
        if key not in self._buffers:
            dev_in = [torch.empty(shape, dtype=torch.int8, device="cuda") for _ in range(2)]
            runs = [self.graph(d, bind=True) for d in dev_in]
            self._buffers[key] = (dev_in, [None, None], runs, torch.cuda.Stream())
        dev_in, dev_out, runs, copy = self._buffers[key]
        ev = lambda: torch.cuda.Event()
        h2d, done, d2h = [ev(), ev()], [ev(), ev()], [ev(), ev()]
        copy.wait_stream(comp)
        with torch.cuda.stream(copy):
            dev_in[0].copy_(host_batches[0], non_blocking=True)
            h2d[0].record(copy)
        for i in range(n):
            j = i % 2
            if i + 1 < n:
                with torch.cuda.stream(copy):
                    if i >= 1:
                        copy.wait_event(done[1 - j])  # step i-1 has finished reading dev_in[1-j]
                    dev_in[1 - j].copy_(host_batches[i + 1], non_blocking=True)
                    h2d[1 - j].record(copy)
            comp.wait_event(h2d[j])
            if i >= 2:
                comp.wait_event(d2h[j])  # dev_out[j] of step i-2 has left the device
            y = runs[j]()
            if post is not None:
                y = post(y)
            if dev_out[j] is None or dev_out[j].shape != y.shape:
                dev_out[j] = torch.empty_like(y)
            dev_out[j].copy_(y, non_blocking=True)
            done[j].record(comp)
            with torch.cuda.stream(copy):
                copy.wait_event(done[j])
                if host_outs[i] is not None:
                    host_outs[i].copy_(dev_out[j], non_blocking=True)
                d2h[j].record(copy)
        comp.wait_stream(copy)

    def _layer_events(self):
        """Four timing events (start, after K1, after K3, end); the middle two
        are re-recorded inside the C ABI (rnsw_conv_forward*_ev), so the
        stage times belong to exactly the kernel chain the untimed call runs."""
        torch = _torch()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        for e in ev[1:3]:
            e.record()  # create the CUDA events (torch creates them lazily)
        handles = (_native.c_void_p * 2)(ev[1]._as_parameter_.value, ev[2]._as_parameter_.value)
        return ev, handles

    def forward_fused_staged(self, x, record):
        """forward_fused() with CUDA events between the kernels of every layer
        (``record(kind, layer, start, end)``): kinds input_transform, gemm or
        product (C <= 4), output_transform (with the fused glue)."""
        l = _native.lib()
        vp = _native.c_void_p
        batch = int(x.shape[0])
        bufs = self._alloc(batch)
        s = _stream_ptr()
        ws = bufs["ws"]
        cur = x.contiguous()
        nl = len(self.cfg.layers)
        for i, ((name, side, c, k, pool), bank) in enumerate(zip(self.cfg.layers, self.banks)):
            oside = side // 2 if pool else side
            nxt = bufs["out"] if i == nl - 1 else \
                bufs["act"][i % 2][: batch * oside * oside * k].view(batch, oside, oside, k)
            ev, handles = self._layer_events()
            ev[0].record()
            _native.check(l.rnsw_conv_forward_requant_ev(self.plan.handle, vp(cur.data_ptr()), batch, side, side, c,
                                                         k, 1, vp(bank.data.data_ptr()), self.cfg.shifts[i],
                                                         1 if pool else 0, vp(nxt.data_ptr()), vp(ws.data_ptr()),
                                                         ws.numel(), s, handles))
            ev[3].record()
            record("input_transform", i, ev[0], ev[1])
            record("product" if c <= 4 else "gemm", i, ev[1], ev[2])
            record("output_transform", i, ev[2], ev[3])
            cur = nxt
        return cur

    def forward(self, x, keep_int32: bool = False, keep_images=None):
        """x: (B, 224, 224, 3) int8 CUDA tensor (NHWC).  Returns the final
        (B, 7, 7, 512) int8 map, plus every layer's int32 output if asked
        (only the images listed in ``keep_images``, when given)."""
        torch = _torch()
        l = _native.lib()
        vp = _native.c_void_p
        batch = int(x.shape[0])
        bufs = self._alloc(batch)
        s = _stream_ptr()
        ws = bufs["ws"]
        cur = x.contiguous()
        outs = []
        nl = len(self.cfg.layers)
        for i, ((name, side, c, k, pool), bank) in enumerate(zip(self.cfg.layers, self.banks)):
            y = bufs["y"][: batch * side * side * k].view(batch, side, side, k)
            _native.check(l.rnsw_conv_forward(self.plan.handle, vp(cur.data_ptr()), batch, side, side, c, k, 1,
                                              _native.LAYOUT_NHWC, vp(bank.data.data_ptr()), vp(y.data_ptr()),
                                              vp(ws.data_ptr()), ws.numel(), s))
            if keep_int32:
                outs.append(y[list(keep_images)].clone() if keep_images is not None else y.clone())
            oside = side // 2 if pool else side
            if i == nl - 1:
                nxt = bufs["out"]
            else:
                nxt = bufs["act"][i % 2][: batch * oside * oside * k].view(batch, oside, oside, k)
            _native.check(l.rnsw_requant_pool(vp(y.data_ptr()), batch, side, side, k, self.cfg.shifts[i],
                                              1 if pool else 0, vp(nxt.data_ptr()), s))
            cur = nxt
        return (cur, outs) if keep_int32 else cur


def direct_ops(batch: int) -> int:
    return workloads.VGGConfig(batch=batch).direct_ops()
