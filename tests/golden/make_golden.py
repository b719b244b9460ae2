"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container, where the reference package is importable
read-only (it is absent on the GPU box, so the fixtures are committed):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden.py

Outputs
  transforms.json   modular AT/G/BT for every (M, R, modulus) the configs and
                    parity cases use, plus compatibility flags
                    (rnswinograd.transforms.reduce_transforms_mod)
  small_cases.npz   seeded small layers: inputs, reference winograd_layer_conv
                    and direct_conv outputs, per-stage outputs
  digests.json      sha256 of inputs / outputs of the full-size BASELINE
                    configs (1, 3, 5 and VGG16 batch 1, every layer) computed
                    by the reference
  scalars.json      known answers: MRC inverses, signed bounds, chunk sizes
  tiles.npz         single-tile API: kernel.tile_conv_mod / rns_tile_conv on
                    seeded (stacked) tiles, 8- and 16-bit moduli
  qtns.json         layer.write_tensor bytes (hex) of seeded int8 / int32 tensors
  vgg_shards.json   config 4 beyond image 0: reference final-map digests for one
                    image per 32-image shard, per-layer int32 digests for two

``--only tiles,qtns`` regenerates just the named fixtures.
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from rnswinograd import gemm, kernel, layer, residue, transforms  # noqa: E402  (the reference)

from paper_2007_12216_b200 import workloads as W  # noqa: E402  (seeded input generation only)

TILES = [(2, 3), (4, 3), (6, 3), (8, 3), (10, 3), (12, 3), (14, 3), (8, 5), (12, 5), (2, 5), (4, 5)]
MODULI = [251, 241, 239, 253, 247, 4001, 4331, 7, 11, 13]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_transforms():
    out = {}
    for m, r in TILES:
        ts = transforms.cached_transforms(m, r)
        for q in MODULI:
            key = f"F{m}x{r}/{q}"
            ok = transforms.check_modulus_compatibility(ts, q)
            ent = {"compatible": bool(ok)}
            if ok:
                mt = transforms.reduce_transforms_mod(ts, q)
                ent.update(at=mt.at.tolist(), g=mt.g.tolist(), bt=mt.bt.tolist(), dtype=str(mt.at.dtype))
            out[key] = ent
    return out


SMALL = [
    # name, h, w, c, k, r, pad, batch, tile_m, moduli, value range
    ("fast1", 8, 8, 3, 5, 3, 1, 2, 4, (251, 241, 239), 128),
    ("fast2", 16, 16, 4, 3, 5, 2, 1, 12, (4001, 4331), 128),
    ("fast3", 30, 30, 7, 2, 3, 0, 1, 14, (251, 241, 239), 128),
    ("fast4", 28, 28, 32, 16, 3, 1, 1, 14, (251, 241, 239), 128),
    ("fast5", 6, 10, 2, 2, 3, 1, 1, 2, (253, 251, 247), 128),
    ("cfg1s", 20, 20, 64, 64, 3, 1, 1, 8, (251, 241, 239), 32),
    ("cfg3s", 15, 13, 24, 40, 5, 2, 2, 8, (251, 241, 239), 16),
    ("vgg16s", 16, 16, 48, 40, 3, 1, 1, 14, (4001, 4331), 128),
    ("small7", 9, 9, 5, 3, 3, 1, 1, 4, (7, 11, 13), 4),
    ("mixed", 12, 12, 12, 20, 3, 1, 1, 10, (251, 4001), 64),
]
STAGE_CASES = {"fast1", "fast2", "fast3", "fast5", "small7", "mixed"}  # per-stage arrays kept small


def gen_small():
    arrays = {}
    meta = []
    for name, h, w, c, k, r, pad, batch, tm, mods, vr in SMALL:
        rng = W.make_rng(2020, f"golden/{name}")
        wt = rng.integers(-vr, vr, (r, r, c, k)).astype(np.int8)
        x = rng.integers(-vr, vr, (batch, h, w, c)).astype(np.int8)
        spec = layer.LayerSpec(h=h, w=w, c=c, k=k, r=r, padding=pad, batch=batch, tile_m=tm)
        system = residue.RnsSystem(mods)
        direct = layer.direct_conv(spec, wt, x)
        rns = layer.winograd_layer_conv(spec, wt, x, system, declared_bound=system.signed_bound)
        arrays[f"{name}/x"] = x
        arrays[f"{name}/w"] = wt
        arrays[f"{name}/direct"] = direct
        arrays[f"{name}/rns"] = rns
        # per-stage outputs (rw/layer.py:266-298) for every modulus
        ts = transforms.cached_transforms(tm, r)
        mts = transforms.reduce_for_system(ts, system)
        patches, _ = layer.tile_decompose(x, tm, r, pad)
        filt = layer.precompute_filter_transforms(wt, mts)
        for mt in (mts if name in STAGE_CASES else ()):
            mm = mt.modulus
            d = kernel.residue_encode_array(patches.transpose(0, 1, 2, 5, 3, 4), mm)
            v = kernel.input_transform_mod(d, mt)
            n = mt.n
            p = patches.shape[0] * patches.shape[1] * patches.shape[2]
            vpos = np.ascontiguousarray(v.transpose(4, 5, 0, 1, 2, 3)).reshape(n * n, p, c)
            acc = layer._modular_gemm(vpos, filt[mm].reshape(n * n, c, k), mm)
            prod = np.ascontiguousarray(acc.reshape(n, n, p, k).transpose(2, 3, 0, 1)).astype(
                gemm.dtype_for_modulus(mm))
            y = kernel.backward_transform_mod(prod, mt)
            arrays[f"{name}/{mm}/U"] = filt[mm]
            arrays[f"{name}/{mm}/V"] = vpos
            arrays[f"{name}/{mm}/acc"] = acc
            arrays[f"{name}/{mm}/y"] = y
        meta.append(dict(name=name, h=h, w=w, c=c, k=k, r=r, pad=pad, batch=batch, tile_m=tm, moduli=list(mods)))
    return arrays, meta


def gen_digests():
    out = {}
    t0 = time.time()
    case, w, x = W.config1()
    spec = layer.LayerSpec(h=case.h, w=case.w, c=case.c, k=case.k, r=case.r, padding=case.pad, batch=case.batch,
                           tile_m=case.tile_m)
    y = layer.winograd_layer_conv(spec, w, x, residue.RnsSystem(case.moduli), declared_bound=case.declared_bound)
    assert np.array_equal(y, layer.direct_conv(spec, w, x))
    out["cfg1"] = dict(x=sha(x), w=sha(w), y=sha(y), ysum=int(y.astype(np.int64).sum()))
    print("cfg1", time.time() - t0, flush=True)

    case, w, x = W.config3()
    spec = layer.LayerSpec(h=case.h, w=case.w, c=case.c, k=case.k, r=case.r, padding=case.pad, batch=case.batch,
                           tile_m=case.tile_m)
    y = layer.winograd_layer_conv(spec, w, x, residue.RnsSystem(case.moduli), declared_bound=case.declared_bound)
    assert np.array_equal(y, layer.direct_conv(spec, w, x))
    out["cfg3"] = dict(x=sha(x), w=sha(w), y=sha(y), ysum=int(y.astype(np.int64).sum()))
    print("cfg3", time.time() - t0, flush=True)

    w, x = W.config5_operands()
    base = layer.LayerSpec(h=28, w=28, c=256, k=256, r=3, padding=1, batch=32)
    direct = layer.direct_conv(base, w, x)
    out["cfg5/direct"] = dict(x=sha(x), w=sha(w), y=sha(direct), ysum=int(direct.astype(np.int64).sum()))
    for case in W.config5_cases():
        spec = layer.LayerSpec(h=28, w=28, c=256, k=256, r=3, padding=1, batch=32, tile_m=case.tile_m)
        y = layer.winograd_layer_conv(spec, w, x, residue.RnsSystem(case.moduli), declared_bound=case.declared_bound)
        assert np.array_equal(y, direct), case.name
        out[case.name] = dict(y=sha(y))
        print(case.name, time.time() - t0, flush=True)

    out.update(gen_vgg_digests())
    return out


def gen_vgg_digests():
    """Config 2: VGG16 batch 1 (image 0), every layer and the final map."""
    t0 = time.time()
    out = {}
    weights = W.vgg16_weights()
    bounds = W.vgg16_bounds(weights)
    x = W.vgg16_images(1)
    out["vgg16/image0"] = dict(x=sha(x))
    system = residue.RnsSystem(W.SYS16)
    for i, ((name, side, c, k, pool), wt) in enumerate(zip(W.VGG16_LAYERS, weights)):
        spec = layer.LayerSpec(h=side, w=side, c=c, k=k, r=3, padding=1, batch=1, tile_m=14)
        y = layer.winograd_layer_conv(spec, wt, x, system, declared_bound=bounds[i])
        d = layer.direct_conv(spec, wt, x)
        assert np.array_equal(y, d), name
        out[f"vgg16/{name}"] = dict(w=sha(wt), y=sha(y), bound=bounds[i], max_abs=int(np.abs(d).max()))
        v = np.clip(np.maximum(y, 0) >> W.VGG16_SHIFTS[i], 0, 127).astype(np.int8)
        if pool:
            b, hh, ww, cc = v.shape
            v = v.reshape(b, hh // 2, 2, ww // 2, 2, cc).max(axis=(2, 4))
        x = np.ascontiguousarray(v)
        print(name, time.time() - t0, flush=True)
    out["vgg16/final"] = dict(y=sha(x))
    return out


VGG_SHARD_IMAGES = (32, 64, 96, 128, 160, 192, 224, 255)  # one per 32-image shard of config 4 (+ the last)
VGG_LAYER_IMAGES = (128, 255)                              # per-layer int32 digests for these


def gen_vgg_shards():
    """Config 4 beyond image 0: the reference RNS path (winograd_layer_conv,
    the declared bounds of workloads.vgg16_bounds) through all 13 layers plus
    the BASELINE glue for one image of every 32-image shard; per-layer int32
    digests for VGG_LAYER_IMAGES (conv4_2..conv5_3 run at the signed bound)."""
    t0 = time.time()
    weights = W.vgg16_weights()
    bounds = W.vgg16_bounds(weights)
    system = residue.RnsSystem(W.SYS16)
    out = {}
    for idx in VGG_SHARD_IMAGES:
        x = W.vgg16_images(1, start=idx)
        rec = {"x": sha(x)}
        for i, ((name, side, c, k, pool), wt) in enumerate(zip(W.VGG16_LAYERS, weights)):
            spec = layer.LayerSpec(h=side, w=side, c=c, k=k, r=3, padding=1, batch=1, tile_m=14)
            y = layer.winograd_layer_conv(spec, wt, x, system, declared_bound=bounds[i])
            if idx in VGG_LAYER_IMAGES:
                rec[name] = sha(y)
            v = np.clip(np.maximum(y, 0) >> W.VGG16_SHIFTS[i], 0, 127).astype(np.int8)
            if pool:
                b, hh, ww, cc = v.shape
                v = v.reshape(b, hh // 2, 2, ww // 2, 2, cc).max(axis=(2, 4))
            x = np.ascontiguousarray(v)
        rec["final"] = sha(x)
        out[str(idx)] = rec
        print("vgg shard image", idx, time.time() - t0, flush=True)
    return out


def gen_verify():
    """The reference's own 217-case verification sweep (rw/cli.py:278-334):
    case list and a digest of every layer_conv output (== direct_conv)."""
    from rnswinograd import cli

    ref_cases = cli.default_verify_cases(2020)
    mine = W.verify_cases(2020)
    assert len(ref_cases) == len(mine)
    out = []
    for rc, mc in zip(ref_cases, mine):
        sp = rc.spec
        assert (sp.tile_m, sp.r, sp.h, sp.w, sp.c, sp.k, sp.padding, sp.batch) == (
            mc["tile_m"], mc["r"], mc["h"], mc["w"], mc["c"], mc["k"], mc["pad"], mc["batch"])
        rng = cli.make_rng(*rc.entropy)
        w = cli.random_int8(rng, sp.weight_shape())
        x = cli.random_int8(rng, sp.input_shape())
        wm, xm = W.verify_operands(mc)
        assert np.array_equal(w, wm) and np.array_equal(x, xm)
        y = layer.layer_conv(sp, w, x, residue.RnsSystem(rc.moduli))
        assert np.array_equal(y, layer.direct_conv(sp, w, x))
        out.append(dict(label=rc.label, y=sha(y)))
    return out


def gen_scalars():
    out = {}
    for mods in [(251, 241, 239), (253, 251, 247), (4001, 4331), (7, 11, 13), (251, 4001)]:
        s = residue.RnsSystem(mods)
        out["x".join(map(str, mods))] = dict(signed_bound=s.signed_bound, dynamic_range=s.dynamic_range,
                                             mrc_inv=s._mrc_inv)
    out["accumulation_chunk"] = {str(m): gemm.accumulation_chunk(m) for m in MODULI if m >= 3}
    out["mod_inverse_14400"] = {str(m): residue.mod_inverse(14400, m) for m in (253, 251, 247)}
    rng = np.random.default_rng(7)
    vals = rng.integers(-7_000_000, 7_000_000, 64)
    s = residue.RnsSystem((251, 241, 239))
    res = [np.array([residue.mod_reduce(int(v), m) for v in vals]) for m in s.moduli]
    out["mrc_251x241x239"] = dict(values=vals.tolist(), residues=[r.tolist() for r in res],
                                  reconstructed=residue.mrc_reconstruct_arrays(res, s).tolist())
    return out


def gen_tiles():
    """kernel.tile_conv_mod on residue tiles and kernel.rns_tile_conv on int8
    tiles, with leading stack dims and a broadcast filter."""
    arrays, meta = {}, []
    cases = [(2, 3, 251, (5,)), (8, 3, 4331, (3, 2)), (4, 5, 241, (4,)), (14, 3, 4001, (2,)), (6, 3, 7, (3,))]
    for i, (m, r, q, lead) in enumerate(cases):
        rng = W.make_rng(2020, "tiles", i)
        n = m + r - 1
        mt = transforms.reduce_transforms_mod(transforms.cached_transforms(m, r), q)
        h = (q - 1) // 2
        g = rng.integers(-h, h + 1, lead + (r, r)).astype(np.int32)
        d = rng.integers(-h, h + 1, lead + (n, n)).astype(np.int32)
        y = kernel.tile_conv_mod(g, d, mt)
        arrays.update({f"mod{i}_g": g, f"mod{i}_d": d, f"mod{i}_y": np.asarray(y)})
        meta.append({"kind": "mod", "i": i, "m": m, "r": r, "modulus": q})
    systems = [(2, 3, (251, 241, 239), (6,), False), (8, 3, (4001, 4331), (2, 3), True), (4, 5, (251, 241, 239), (3,), False)]
    for i, (m, r, mods, lead, bcast) in enumerate(systems):
        rng = W.make_rng(2020, "rns_tiles", i)
        n = m + r - 1
        system = residue.RnsSystem(mods)
        mts = transforms.reduce_for_system(transforms.cached_transforms(m, r), system)
        g = rng.integers(-128, 128, ((r, r) if bcast else lead + (r, r))).astype(np.int8)
        d = rng.integers(-128, 128, lead + (n, n)).astype(np.int8)
        y = kernel.rns_tile_conv(g, d, system, mts)
        arrays.update({f"rns{i}_g": g, f"rns{i}_d": d, f"rns{i}_y": np.asarray(y)})
        meta.append({"kind": "rns", "i": i, "m": m, "r": r, "moduli": list(mods)})
    return arrays, meta


def gen_qtns(tmp: Path):
    out = []
    rng = W.make_rng(2020, "qtns")
    tensors = [rng.integers(-128, 128, (2, 3, 4, 5)).astype(np.int8),
               rng.integers(-2**31, 2**31, (3, 7)).astype(np.int32),
               np.array(-5, dtype=np.int32), np.zeros((0, 4), dtype=np.int8)]
    for i, a in enumerate(tensors):
        path = tmp / f"t{i}.qtns"
        layer.write_tensor(path, a)
        out.append({"dtype": str(a.dtype), "shape": list(a.shape), "values": a.reshape(-1).tolist(),
                    "bytes_hex": path.read_bytes().hex()})
    return out


def main():
    if "--only" in sys.argv:
        only = set(sys.argv[sys.argv.index("--only") + 1].split(","))
        if "tiles" in only:
            arrays, meta = gen_tiles()
            np.savez_compressed(HERE / "tiles.npz", **arrays)
            (HERE / "tiles.json").write_text(json.dumps(meta, indent=1))
        if "vggdigests" in only:
            d = json.loads((HERE / "digests.json").read_text())
            d = {k: v for k, v in d.items() if not k.startswith("vgg16/")}
            d.update(gen_vgg_digests())
            (HERE / "digests.json").write_text(json.dumps(d, indent=1))
        if "vggshards" in only:
            (HERE / "vgg_shards.json").write_text(json.dumps(gen_vgg_shards(), indent=1))
        if "qtns" in only:
            import tempfile

            with tempfile.TemporaryDirectory() as td:
                (HERE / "qtns.json").write_text(json.dumps(gen_qtns(Path(td)), indent=0))
        return
    (HERE / "transforms.json").write_text(json.dumps(gen_transforms()))
    (HERE / "scalars.json").write_text(json.dumps(gen_scalars(), indent=1))
    arrays, meta = gen_small()
    np.savez_compressed(HERE / "small_cases.npz", **arrays)
    (HERE / "small_cases.json").write_text(json.dumps(meta, indent=1))
    (HERE / "verify.json").write_text(json.dumps(gen_verify(), indent=0))
    arrays, meta = gen_tiles()
    np.savez_compressed(HERE / "tiles.npz", **arrays)
    (HERE / "tiles.json").write_text(json.dumps(meta, indent=1))
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        (HERE / "qtns.json").write_text(json.dumps(gen_qtns(Path(td)), indent=0))
    if "--no-digests" not in sys.argv:
        (HERE / "digests.json").write_text(json.dumps(gen_digests(), indent=1))


if __name__ == "__main__":
    main()
