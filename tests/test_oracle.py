"""The CPU oracle (oracle/ref_port.py, oracle/oracle.c) against golden vectors
produced by the reference itself.  Runs without a GPU."""
import numpy as np
import pytest

import oracle
from oracle import ref_port as O
from oracle.vgg_ref import requant_pool
from golden_util import digests, sha, small_arrays, small_meta, scalars, transforms


def test_modular_matrices_match_reference_golden():
    gold = transforms()
    checked = 0
    for key, ent in gold.items():
        if not ent["compatible"]:
            continue
        fm, mod = key.split("/")
        m_out, r = (int(v) for v in fm[1:].split("x"))
        at, g, bt = O.modular_matrices(m_out, r, int(mod))
        assert at.tolist() == ent["at"] and g.tolist() == ent["g"] and bt.tolist() == ent["bt"], key
        assert str(at.dtype) == ent["dtype"]
        checked += 1
    assert checked > 60


@pytest.mark.parametrize("meta", small_meta(), ids=lambda m: m["name"])
def test_layer_port_matches_reference(meta):
    a = small_arrays()
    n = meta["name"]
    x, w = a[f"{n}/x"], a[f"{n}/w"]
    got = O.winograd_layer(x, w, meta["pad"], meta["tile_m"], tuple(meta["moduli"]))
    assert got.dtype == np.int32
    assert np.array_equal(got, a[f"{n}/rns"])
    assert np.array_equal(O.direct_conv(x, w, meta["pad"]), a[f"{n}/direct"])
    assert np.array_equal(oracle.direct_conv_c(x, w, meta["pad"]), a[f"{n}/direct"])


@pytest.mark.parametrize("meta", [m for m in small_meta() if f"{m['name']}/{m['moduli'][0]}/V" in small_arrays()],
                         ids=lambda m: m["name"])
def test_stage_functions_match_reference(meta):
    a = small_arrays()
    n = meta["name"]
    x, w = a[f"{n}/x"], a[f"{n}/w"]
    patches, _ = O.patches_of(x, meta["tile_m"], meta["r"], meta["pad"])
    for m in meta["moduli"]:
        at, g, bt = O.modular_matrices(meta["tile_m"], meta["r"], m)
        mats = {m: (at, g, bt)}
        u = O.filter_bank(w, mats)[m]
        assert np.array_equal(u, a[f"{n}/{m}/U"])
        assert np.array_equal(O.filter_bank_fast(w, mats)[m], u)
        v = O.input_stage(patches, bt, m)
        assert np.array_equal(v, a[f"{n}/{m}/V"])
        acc = O.gemm_stage(v, u, m)
        assert np.array_equal(acc, a[f"{n}/{m}/acc"])
        assert np.array_equal(O.output_stage(acc, at, m), a[f"{n}/{m}/y"])


def test_mrc_matches_reference():
    s = scalars()["mrc_251x241x239"]
    res = [np.array(r) for r in s["residues"]]
    assert O.mrc(res, (251, 241, 239)).tolist() == s["reconstructed"] == s["values"]


def test_chunk_lengths_match_reference():
    for m, v in scalars()["accumulation_chunk"].items():
        assert O.chunk_len(int(m)) == v


def test_c_oracle_sandwich_and_mrc_scalars():
    import ctypes

    lib = oracle.lib()
    at, g, bt = O.modular_matrices(4, 3, 251)
    rng = np.random.default_rng(3)
    d = rng.integers(-125, 126, (6, 6)).astype(np.int32)
    L = np.ascontiguousarray(bt, dtype=np.int32)
    R = np.ascontiguousarray(bt.T, dtype=np.int32)
    out = np.empty((6, 6), dtype=np.int32)
    lib.oracle_sandwich_mod(L.ctypes.data, d.ctypes.data, R.ctypes.data, 6, 6, 6, 6, 251, out.ctypes.data)
    assert np.array_equal(out, O.sandwich(bt, d, bt.T, 251))
    mods = np.array([4001, 4331], dtype=np.int32)
    for v in (0, 1, -1, 8664165, -8664165, 123456, -7654321):
        r = np.array([O.sym(v, 4001), O.sym(v, 4331)], dtype=np.int32)
        assert lib.oracle_mrc(r.ctypes.data, mods.ctypes.data, 2) == v


def test_direct_conv_c_edge_shapes():
    rng = np.random.default_rng(11)
    for (b, h, w, c, k, r, pad) in [(1, 1, 1, 1, 1, 1, 0), (2, 5, 3, 7, 4, 3, 2), (1, 9, 9, 3, 2, 5, 0),
                                    (3, 4, 6, 16, 9, 3, 1)]:
        x = rng.integers(-128, 128, (b, h, w, c)).astype(np.int8)
        wt = rng.integers(-128, 128, (r, r, c, k)).astype(np.int8)
        assert np.array_equal(oracle.direct_conv_c(x, wt, pad), O.direct_conv(x, wt, pad))


def test_vgg_glue_restatement():
    rng = np.random.default_rng(5)
    y = rng.integers(-(1 << 20), 1 << 20, (2, 6, 7, 5)).astype(np.int32)
    got = requant_pool(y, 9, True)
    assert got.shape == (2, 3, 3, 5) and got.dtype == np.int8
    v = np.clip(np.maximum(y, 0) >> 9, 0, 127)
    assert got[1, 2, 1, 3] == v[1, 4:6, 2:4, 3].max()


def test_config1_oracle_matches_reference_digest():
    from paper_2007_12216_b200 import workloads as W

    case, w, x = W.config1()
    d = digests()["cfg1"]
    assert sha(x) == d["x"] and sha(w) == d["w"]
    y = O.winograd_layer(x, w, case.pad, case.tile_m, case.moduli)
    assert sha(y) == d["y"]


def test_verify_sweep_generation_and_oracle_sample():
    """Case generation restates rw/cli.py:278-314 (checked against the
    reference in make_golden); the oracle port reproduces a sample."""
    import json

    from golden_util import GOLDEN
    from paper_2007_12216_b200 import workloads as W

    gold = json.loads((GOLDEN / "verify.json").read_text())
    cases = W.verify_cases(2020)
    assert len(cases) == 217
    for idx in range(0, 217, 23):
        c = cases[idx]
        w, x = W.verify_operands(c)
        y = O.winograd_layer(x, w, c["pad"], c["tile_m"], c["moduli"])
        assert sha(y) == gold[idx]["y"], gold[idx]["label"]
