"""GPU side of the single-tile API and the CLI: the reference's own
tile_conv_mod / rns_tile_conv outputs (tests/golden/tiles.npz), the exact
direct correlation, and `verify` / `bench` end to end on the device."""
import csv
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from oracle import ref_port as O

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def _rnsw():
    import paper_2007_12216_b200 as rnsw

    return rnsw


def test_single_tile_api_matches_reference_outputs():
    rnsw = _rnsw()
    meta = json.loads((GOLDEN / "tiles.json").read_text())
    a = np.load(GOLDEN / "tiles.npz")
    for c in meta:
        i, m, r = c["i"], c["m"], c["r"]
        ts = rnsw.cached_transforms(m, r)
        if c["kind"] == "mod":
            mt = rnsw.reduce_transforms_mod(ts, c["modulus"])
            got = rnsw.tile_conv_mod(a[f"mod{i}_g"], a[f"mod{i}_d"], mt)
            assert np.array_equal(got, a[f"mod{i}_y"]), c
        else:
            system = rnsw.RnsSystem(tuple(c["moduli"]))
            got = rnsw.rns_tile_conv(a[f"rns{i}_g"], a[f"rns{i}_d"], system, rnsw.reduce_for_system(ts, system))
            assert got.dtype == np.int32 and np.array_equal(got, a[f"rns{i}_y"]), c


def test_rns_tile_conv_is_the_exact_correlation():
    rnsw = _rnsw()
    rng = np.random.default_rng(3)
    system = rnsw.RnsSystem((4001, 4331))
    m, r = 14, 3
    mts = rnsw.reduce_for_system(rnsw.cached_transforms(m, r), system)
    g = rng.integers(-128, 128, (7, r, r)).astype(np.int8)
    d = rng.integers(-128, 128, (7, m + r - 1, m + r - 1)).astype(np.int8)
    got = rnsw.rns_tile_conv(g, d, system, mts)
    for s in range(7):
        want = oracle.direct_conv_c(d[s][None, :, :, None], g[s][:, :, None, None], 0)[0, :, :, 0]
        assert np.array_equal(got[s], want)


def test_tile_conv_mod_large_modulus_generic_path():
    """A 16-bit modulus above the fast-path range (m >= 4500) runs the generic kernels."""
    rnsw = _rnsw()
    rng = np.random.default_rng(4)
    q, m, r = 8191, 4, 3
    mt = rnsw.reduce_transforms_mod(rnsw.cached_transforms(m, r), q)
    g = rng.integers(-(q // 2), q // 2 + 1, (3, r, r))
    d = rng.integers(-(q // 2), q // 2 + 1, (3, m + r - 1, m + r - 1))
    assert np.array_equal(rnsw.tile_conv_mod(g, d, mt), O.tile_conv_mod(g, d, m, r, q))


def test_cli_verify_file_mode_roundtrip(tmp_path, capsys):
    rnsw = _rnsw()
    from paper_2007_12216_b200 import cli

    rng = np.random.default_rng(5)
    x = rng.integers(-128, 128, (2, 20, 18, 5)).astype(np.int8)
    w = rng.integers(-128, 128, (3, 3, 5, 7)).astype(np.int8)
    rnsw.write_tensor(tmp_path / "x.qtns", x)
    rnsw.write_tensor(tmp_path / "w.qtns", w)
    rc = cli.main(["verify", "--input", str(tmp_path / "x.qtns"), "--weights", str(tmp_path / "w.qtns"),
                   "--output", str(tmp_path / "y.qtns"), "--tile", "6", "--padding", "1"])
    assert rc == 0 and "PASS" in capsys.readouterr().out
    assert np.array_equal(rnsw.read_tensor(tmp_path / "y.qtns"), oracle.direct_conv_c(x, w, 1))


def test_cli_verify_config_and_bench_csv(tmp_path, capsys):
    from paper_2007_12216_b200 import cli

    cfg = {"rns": [251, 241, 239], "tile_m": 6, "iterations": 2, "declared_bound": 200000,
           "layers": [{"name": "small", "h": 12, "w": 12, "c": 3, "k": 8, "r": 3, "padding": 1},
                      {"name": "mid", "h": 14, "w": 14, "c": 32, "k": 16, "r": 3, "padding": 1},
                      {"name": "dir", "h": 10, "w": 10, "c": 16, "k": 16, "r": 3, "padding": 1,
                       "algorithm": "direct"}]}
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(cfg))
    assert cli.main(["verify", "--config", str(path)]) == 0
    out = capsys.readouterr().out
    assert "2/2 cases passed" in out
    assert cli.main(["bench", "--config", str(path), "--csv", str(tmp_path / "b.csv")]) == 0
    out = capsys.readouterr().out
    assert "total" in out and "exact" in out
    rows = list(csv.DictReader(open(tmp_path / "b.csv")))
    assert [r["layer"] for r in rows] == ["small", "mid", "dir"] and all(r["exact"] == "1" for r in rows)
    assert float(rows[1]["gemm_pct"]) > 0 and float(rows[0]["rns_ms"]) > 0


def test_cli_verify_default_sweep_subset(capsys):
    """The default sweep is the reference's 217-case verify (tests/test_gpu_verify.py
    runs all of them); here the CLI prints its summary line."""
    from paper_2007_12216_b200 import cli

    assert cli.main(["verify", "--seed", "2020"]) == 0
    assert "217/217 cases passed" in capsys.readouterr().out
