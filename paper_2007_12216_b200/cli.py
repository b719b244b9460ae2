"""Command line, backed by the GPU path (rw/cli.py ``verify`` / ``bench``).

    python -m paper_2007_12216_b200 verify [--seed S] [--config CFG]
    python -m paper_2007_12216_b200 verify --input X.qtns --weights W.qtns [--output Y.qtns]
                                    [--tile M] [--padding P] [--moduli a,b,c] [--declared-bound D]
    python -m paper_2007_12216_b200 bench [--config CFG] [--csv OUT] [--iterations N] [--seed S]

``verify`` compares the RNS-Winograd layer (``layer_conv``) with an exact
direct convolution on the same GPU: the tcgen05 direct conv where it applies
(C % 16 == 0), otherwise a float64 convolution, which is exact here (every
partial sum is an integer below 2^53).  ``bench`` times both per layer with
CUDA events and prints the reference's table / CSV columns
(rw/cli.py:505-570).  Config files use the reference's JSON schema
(rw/cli.py:105-185), so the reference's own config files load unchanged.
Exit status: 0 all exact, 2 a mismatch, 1 a usage/config error.
"""

from __future__ import annotations

import argparse
import csv
import json
import sys
from dataclasses import dataclass, replace
from fractions import Fraction

import numpy as np

from . import workloads as W
from .errors import DynamicRangeExceeded
from .layer import (LayerSpec, StageTimings, count_operations, direct_conv, layer_conv,
                    precompute_filter_transforms, range_check, winograd_layer_conv)
from .residue import RnsSystem
from .tensor_io import read_tensor, write_tensor
from .transforms import cached_transforms, reduce_for_system

DEFAULT_SEED = W.DEFAULT_SEED


class ConfigError(ValueError):
    """A bad config file or argument combination (rw/cli.py:33-38)."""


def parse_moduli(text: str) -> tuple[int, ...]:
    try:
        mods = tuple(int(t) for t in text.split(",") if t.strip())
    except ValueError:
        raise ConfigError(f"bad moduli list {text!r}") from None
    if not mods:
        raise ConfigError("empty moduli list")
    return mods


# ---------------------------------------------------------------------------
# configs (same JSON schema as the reference)


@dataclass(frozen=True)
class LayerEntry:
    name: str
    spec: LayerSpec
    algorithm: str = "winograd"
    declared_bound: int | None = None


@dataclass(frozen=True)
class BenchConfig:
    rns: tuple[int, ...]
    tile_m: int
    seed: int
    iterations: int
    layers: tuple[LayerEntry, ...]
    declared_bound: int | None = None


def config_from_dict(doc: dict, where: str = "config") -> BenchConfig:
    try:
        rns = tuple(int(m) for m in doc["rns"])
        tile_m = int(doc.get("tile_m", 14))
        seed = int(doc.get("seed", DEFAULT_SEED))
        iterations = int(doc.get("iterations", 1))
        top_bound = doc.get("declared_bound")
        layers = []
        for ent in doc["layers"]:
            algorithm = ent.get("algorithm", "winograd")
            if algorithm not in ("winograd", "direct"):
                raise ConfigError(f"{where}: layer {ent.get('name')!r} has unknown algorithm {algorithm!r}")
            spec = LayerSpec(h=int(ent["h"]), w=int(ent["w"]), c=int(ent["c"]), k=int(ent["k"]), r=int(ent["r"]),
                             batch=int(ent.get("batch", 1)), padding=int(ent.get("padding", 0)),
                             stride=int(ent.get("stride", 1)), tile_m=int(ent.get("tile_m", tile_m)))
            layers.append(LayerEntry(name=str(ent.get("name", f"layer{len(layers)}")), spec=spec,
                                     algorithm=algorithm, declared_bound=ent.get("declared_bound", top_bound)))
    except ConfigError:
        raise
    except (KeyError, TypeError, ValueError) as e:
        raise ConfigError(f"{where}: {e!r}") from None
    if not layers:
        raise ConfigError(f"{where}: no layers")
    if iterations < 1:
        raise ConfigError(f"{where}: iterations must be >= 1")
    return BenchConfig(rns=rns, tile_m=tile_m, seed=seed, iterations=iterations, layers=tuple(layers),
                       declared_bound=top_bound)


def load_config(path) -> BenchConfig:
    try:
        with open(path) as f:
            doc = json.load(f)
    except OSError as e:
        raise ConfigError(f"cannot read config {path}: {e}") from None
    except json.JSONDecodeError as e:
        raise ConfigError(f"config {path} is not valid JSON: {e}") from None
    return config_from_dict(doc, str(path))


def default_config() -> BenchConfig:
    """The 13 VGG16 3x3 layers at batch 1 (workloads.VGG16_LAYERS), F(14,3)
    over RNS(4001, 4331): BASELINE config 2 without the inter-layer glue."""
    layers = [{"name": name, "h": side, "w": side, "c": c, "k": k, "r": 3, "padding": 1}
              for name, side, c, k, _pool in W.VGG16_LAYERS]
    return config_from_dict({"rns": list(W.SYS16), "tile_m": 14, "seed": DEFAULT_SEED, "layers": layers},
                            "default VGG16 config")


# ---------------------------------------------------------------------------
# exact GPU comparator


def exact_direct(spec: LayerSpec, weights, x):
    """Exact int32 direct convolution on the GPU (torch tensors in and out)."""
    import torch
    import torch.nn.functional as F

    if spec.c % 16 == 0:
        return direct_conv(spec, weights, x)
    xd = torch.as_tensor(x).cuda().permute(0, 3, 1, 2).to(torch.float64)
    wd = torch.as_tensor(weights).cuda().permute(3, 2, 0, 1).to(torch.float64)
    y = F.conv2d(xd, wd, padding=spec.padding, stride=spec.stride)
    return y.round().to(torch.int32).permute(0, 2, 3, 1).contiguous()


def _to_numpy(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def _first_mismatch(want: np.ndarray, got: np.ndarray):
    bad = np.argwhere(want != got)
    first = tuple(int(v) for v in bad[0])
    return len(bad), first


# ---------------------------------------------------------------------------
# verify


def _verify_one(label: str, spec: LayerSpec, moduli, weights, x, declared_bound) -> tuple[bool, str]:
    import torch

    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(weights).cuda()
    want = _to_numpy(exact_direct(spec, wd, xd))
    got = _to_numpy(layer_conv(spec, wd, xd, RnsSystem(moduli), declared_bound=declared_bound))
    if np.array_equal(want, got):
        return True, f"PASS {label}"
    n, first = _first_mismatch(want, got)
    return False, f"FAIL {label} mismatches={n} first at {first}: got {int(got[first])}, want {int(want[first])}"


def cmd_verify(args) -> int:
    if args.input or args.weights:
        if not (args.input and args.weights):
            raise ConfigError("file mode needs both --input and --weights")
        return _verify_files(args)
    seed = args.seed if args.seed is not None else DEFAULT_SEED
    runs = []  # (label, spec, moduli, weights, x, declared_bound)
    if args.config:
        cfg = load_config(args.config)
        seed = args.seed if args.seed is not None else cfg.seed
        for ent in cfg.layers:
            if ent.algorithm != "winograd":
                continue
            rng = W.make_rng(seed, ent.name)
            w = W.uniform_int8(rng, ent.spec.weight_shape(), -128, 127)
            x = W.uniform_int8(rng, ent.spec.input_shape(), -128, 127)
            runs.append((f"{ent.name} rns={cfg.rns}", ent.spec, cfg.rns, w, x, ent.declared_bound))
        if not runs:
            raise ConfigError(f"{args.config}: no winograd layers to verify")
    else:
        for case in W.verify_cases(seed):
            w, x = W.verify_operands(case)
            spec = LayerSpec(h=case["h"], w=case["w"], c=case["c"], k=case["k"], r=case["r"], batch=case["batch"],
                             padding=case["pad"], tile_m=case["tile_m"])
            label = (f"F({case['tile_m']}x{case['tile_m']},{case['r']}x{case['r']}) rns={case['moduli']} "
                     f"h={case['h']} w={case['w']} c={case['c']} k={case['k']} pad={case['pad']} b={case['batch']}")
            runs.append((label, spec, case["moduli"], w, x, None))
    failures = 0
    for label, spec, moduli, w, x, bound in runs:
        try:
            ok, line = _verify_one(label, spec, moduli, w, x, bound)
        except DynamicRangeExceeded as e:
            rep = range_check(spec, RnsSystem(moduli), bound)
            print(f"FAIL {label} dynamic range: {e}")
            print(f"     static bound {rep.static_bound}, declared {rep.declared_bound}, "
                  f"signed bound {rep.signed_bound}")
            failures += 1
            continue
        print(line)
        failures += 0 if ok else 1
    print(f"{len(runs) - failures}/{len(runs)} cases passed")
    return 0 if failures == 0 else 2


def _verify_files(args) -> int:
    import torch

    x = read_tensor(args.input)
    weights = read_tensor(args.weights)
    if weights.ndim != 4 or x.ndim != 4:
        raise ConfigError("tensors must be rank 4: input NHWC, weights (r, r, c, k)")
    r, r2, c, k = weights.shape
    if r != r2 or x.shape[3] != c:
        raise ConfigError(f"weights {weights.shape} do not describe square filters on {x.shape[3]} input channels")
    spec = LayerSpec(h=x.shape[1], w=x.shape[2], c=c, k=k, r=r, batch=x.shape[0], padding=args.padding,
                     tile_m=args.tile)
    system = RnsSystem(parse_moduli(args.moduli))
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(weights).cuda()
    want = _to_numpy(exact_direct(spec, wd, xd))
    got = _to_numpy(winograd_layer_conv(spec, wd, xd, system, declared_bound=args.declared_bound))
    if args.output:
        write_tensor(args.output, got)
    if np.array_equal(want, got):
        print(f"PASS {args.input} * {args.weights}: outputs match direct conv")
        return 0
    n, first = _first_mismatch(want, got)
    print(f"FAIL {args.input} * {args.weights}: {n} mismatches, first at {first}: "
          f"got {int(got[first])}, want {int(want[first])}")
    return 2


# ---------------------------------------------------------------------------
# bench


@dataclass
class BenchRow:
    name: str
    algorithm: str
    spec: LayerSpec
    direct_ms: float
    rns_ms: float
    timings: StageTimings
    reduction: Fraction
    exact: bool

    @property
    def speedup(self) -> float:
        return self.direct_ms / self.rns_ms if self.rns_ms else float("nan")


def _timed(fn, iterations: int):
    """Best-of-N device time (CUDA events around the call) and the last result."""
    import torch

    best, out = float("inf"), None
    for _ in range(iterations):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best, out


def run_bench(cfg: BenchConfig) -> list[BenchRow]:
    import torch

    system = RnsSystem(cfg.rns)
    rows = []
    children = np.random.SeedSequence(cfg.seed).spawn(len(cfg.layers))
    for ent, child in zip(cfg.layers, children):
        rng = np.random.Generator(np.random.PCG64(child))
        w = rng.integers(-128, 128, ent.spec.weight_shape(), dtype=np.int8)
        x = rng.integers(-128, 128, ent.spec.input_shape(), dtype=np.int8)
        wd, xd = torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda()
        exact_direct(ent.spec, wd, xd)  # warm-up (lazy module loading)
        direct_ms, want = _timed(lambda: exact_direct(ent.spec, wd, xd), cfg.iterations)
        timings = StageTimings()
        if ent.algorithm == "direct":
            rns_ms, got = direct_ms, want
        else:
            # filter transforms depend only on the weights: precomputed outside
            # the timed region, as in the reference bench (rw/cli.py:459-463)
            filters = precompute_filter_transforms(wd, reduce_for_system(
                cached_transforms(ent.spec.tile_m, ent.spec.r), system))
            run = lambda t=None: winograd_layer_conv(ent.spec, wd, xd, system, declared_bound=ent.declared_bound,
                                                     filters=filters, timings=t)
            run()  # warm-up
            rns_ms, got = _timed(run, cfg.iterations)
            run(timings)  # per-stage CUDA-event split of one more call
        rows.append(BenchRow(name=ent.name, algorithm=ent.algorithm, spec=ent.spec, direct_ms=direct_ms,
                             rns_ms=rns_ms, timings=timings,
                             reduction=count_operations(ent.spec, system).reduction_ratio,
                             exact=bool(torch.equal(want, got))))
    return rows


def _pcts(row: BenchRow) -> tuple[float, ...]:
    """Stage shares: tiling, input, gemm, backward, mrc, scatter (rw/cli.py:489-502).
    On the device tiling is part of the input transform and MRC + scatter are
    fused into the backward transform, so those columns read 0."""
    t = row.timings
    total = t.total()
    if total <= 0 or row.algorithm == "direct":
        return (0.0,) * 6
    return tuple(100.0 * v / total for v in (t.tiling, t.input_transform, t.gemm, t.backward_transform, t.mrc,
                                             t.scatter))


def cmd_bench(args) -> int:
    cfg = load_config(args.config) if args.config else default_config()
    if args.iterations is not None:
        cfg = replace(cfg, iterations=args.iterations)
    if args.seed is not None:
        cfg = replace(cfg, seed=args.seed)
    if cfg.iterations < 1:
        raise ConfigError("iterations must be >= 1")
    rows = run_bench(cfg)
    print(f"rns={cfg.rns}  tile_m={cfg.tile_m}  seed={cfg.seed}  iterations={cfg.iterations}  (B200, CUDA events)")
    print("filter transforms are precomputed per layer and excluded from rns ms")
    header = (f"{'layer':<10} {'alg':<8} {'direct ms':>10} {'rns ms':>10} {'speedup':>8} {'mult red':>9} "
              f"{'tile%':>6} {'inp%':>6} {'gemm%':>6} {'bwd%':>6} {'mrc%':>6} {'scat%':>6}  exact")
    print(header)
    print("-" * len(header))
    for row in rows:
        p = _pcts(row)
        print(f"{row.name:<10} {row.algorithm:<8} {row.direct_ms:>10.3f} {row.rns_ms:>10.3f} {row.speedup:>8.2f} "
              f"{float(row.reduction):>9.2f} " + " ".join(f"{v:>6.1f}" for v in p) + f"  {row.exact}")
    td, tr = sum(r.direct_ms for r in rows), sum(r.rns_ms for r in rows)
    print(f"{'total':<10} {'':<8} {td:>10.3f} {tr:>10.3f} {td / tr if tr else float('nan'):>8.2f}")
    if args.csv:
        with open(args.csv, "w", newline="") as f:
            wr = csv.writer(f)
            wr.writerow(["layer", "algorithm", "h", "w", "c", "k", "r", "direct_ms", "rns_ms", "speedup",
                         "mult_reduction", "tiling_pct", "input_transform_pct", "gemm_pct", "backward_pct",
                         "mrc_pct", "scatter_pct", "exact"])
            for row in rows:
                wr.writerow([row.name, row.algorithm, row.spec.h, row.spec.w, row.spec.c, row.spec.k, row.spec.r,
                             f"{row.direct_ms:.3f}", f"{row.rns_ms:.3f}", f"{row.speedup:.4f}",
                             f"{float(row.reduction):.4f}"] + [f"{v:.2f}" for v in _pcts(row)] + [int(row.exact)])
    return 0 if all(r.exact for r in rows) else 2


# ---------------------------------------------------------------------------


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2007_12216_b200",
                                 description="Exact INT8 convolution by RNS-Winograd on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("verify", help="compare the fast path against direct convolution (GPU)")
    p.add_argument("--seed", type=int, default=None)
    p.add_argument("--config", help="verify the layers of a bench config")
    p.add_argument("--input", help="QTNS int8 input tensor (NHWC)")
    p.add_argument("--weights", help="QTNS int8 weight tensor (r, r, c, k)")
    p.add_argument("--output", help="write the verified output tensor here")
    p.add_argument("--tile", type=int, default=14, help="tile size for file mode")
    p.add_argument("--padding", type=int, default=0, help="padding for file mode")
    p.add_argument("--moduli", default="251,241,239", help="moduli for file mode")
    p.add_argument("--declared-bound", type=int, default=None)
    p.set_defaults(fn=cmd_verify)
    p = sub.add_parser("bench", help="timed sweep over a layer config (GPU)")
    p.add_argument("--config", help="JSON layer config (default: VGG16 3x3 layers, batch 1)")
    p.add_argument("--csv", help="also write results to this CSV file")
    p.add_argument("--iterations", type=int, default=None)
    p.add_argument("--seed", type=int, default=None)
    p.set_defaults(fn=cmd_bench)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except ConfigError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
