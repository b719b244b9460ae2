"""Host side of the CLI / file-format / single-tile surface (no GPU):
QTNS byte parity with the reference's writer, config parsing, argument
errors, and the oracle restatement of the single-tile API pinned to the
reference's own outputs (tests/golden/tiles.npz)."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2007_12216_b200 as rnsw
from paper_2007_12216_b200 import cli
from oracle import ref_port as O

GOLDEN = Path(__file__).resolve().parent / "golden"


def _qtns_cases():
    return json.loads((GOLDEN / "qtns.json").read_text())


@pytest.mark.parametrize("case", _qtns_cases(), ids=lambda c: f"{c['dtype']}{c['shape']}")
def test_qtns_bytes_match_reference_writer(case, tmp_path):
    a = np.array(case["values"], dtype=case["dtype"]).reshape(case["shape"])
    path = tmp_path / "t.qtns"
    rnsw.write_tensor(path, a)
    assert path.read_bytes().hex() == case["bytes_hex"]
    back = rnsw.read_tensor(path)
    assert back.dtype == a.dtype and back.shape == a.shape and np.array_equal(back, a)


def test_qtns_rejects_bad_files(tmp_path):
    p = tmp_path / "bad.qtns"
    p.write_bytes(b"NOPE\x01\x00\x08")
    with pytest.raises(ValueError, match="not a QTNS"):
        rnsw.read_tensor(p)
    good = tmp_path / "g.qtns"
    rnsw.write_tensor(good, np.arange(6, dtype=np.int8).reshape(2, 3))
    raw = bytearray(good.read_bytes())
    raw[4] = 2  # version
    p.write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="version"):
        rnsw.read_tensor(p)
    raw = bytearray(good.read_bytes())
    raw[6 + 4 * 2] = 16  # element width
    p.write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="width"):
        rnsw.read_tensor(p)
    p.write_bytes(good.read_bytes()[:-1])
    with pytest.raises(ValueError, match="payload"):
        rnsw.read_tensor(p)
    with pytest.raises(rnsw.ShapeMismatch):
        rnsw.write_tensor(p, np.zeros(3, dtype=np.int16))


def test_config_parsing_and_errors(tmp_path):
    cfg = cli.config_from_dict({"rns": [251, 241, 239], "declared_bound": 1000,
                                "layers": [{"name": "a", "h": 8, "w": 9, "c": 3, "k": 4, "r": 3, "padding": 1},
                                           {"h": 8, "w": 8, "c": 16, "k": 4, "r": 3, "algorithm": "direct",
                                            "declared_bound": 5}]})
    assert cfg.tile_m == 14 and cfg.seed == cli.DEFAULT_SEED and cfg.iterations == 1
    assert cfg.layers[0].declared_bound == 1000 and cfg.layers[1].declared_bound == 5
    assert cfg.layers[1].name == "layer1" and cfg.layers[1].algorithm == "direct"
    for bad in ({"layers": []}, {"rns": [7], "layers": []}, {"rns": [7], "layers": [{"h": 1}]},
                {"rns": [7], "iterations": 0, "layers": [{"h": 4, "w": 4, "c": 1, "k": 1, "r": 3}]},
                {"rns": [7], "layers": [{"h": 4, "w": 4, "c": 1, "k": 1, "r": 3, "algorithm": "fft"}]}):
        with pytest.raises(cli.ConfigError):
            cli.config_from_dict(bad)
    with pytest.raises(cli.ConfigError):
        cli.load_config(tmp_path / "missing.json")
    (tmp_path / "x.json").write_text("{not json")
    with pytest.raises(cli.ConfigError):
        cli.load_config(tmp_path / "x.json")
    d = cli.default_config()
    assert [e.name for e in d.layers][:2] == ["conv1_1", "conv1_2"] and d.rns == (4001, 4331)
    assert cli.parse_moduli("251, 241,239") == (251, 241, 239)
    with pytest.raises(cli.ConfigError):
        cli.parse_moduli("a,b")


def test_cli_usage_errors_before_device_work(capsys):
    assert cli.main(["verify", "--input", "only.qtns"]) == 1
    assert "both --input and --weights" in capsys.readouterr().err
    with pytest.raises(SystemExit):
        cli.main(["frobnicate"])


def _tile_cases():
    meta = json.loads((GOLDEN / "tiles.json").read_text())
    arrays = np.load(GOLDEN / "tiles.npz")
    return meta, arrays


def test_oracle_single_tile_api_matches_reference():
    meta, a = _tile_cases()
    for c in meta:
        i = c["i"]
        if c["kind"] == "mod":
            got = O.tile_conv_mod(a[f"mod{i}_g"], a[f"mod{i}_d"], c["m"], c["r"], c["modulus"])
            assert np.array_equal(got, a[f"mod{i}_y"]), c
        else:
            got = O.rns_tile_conv(a[f"rns{i}_g"], a[f"rns{i}_d"], c["m"], c["r"], tuple(c["moduli"]))
            assert np.array_equal(got, a[f"rns{i}_y"]), c


def test_tile_api_host_checks_raise_before_device_work():
    system = rnsw.RnsSystem((251, 241, 239))
    mts = rnsw.reduce_for_system(rnsw.cached_transforms(4, 3), system)
    g, d = np.zeros((3, 3), np.int8), np.zeros((6, 6), np.int8)
    with pytest.raises(rnsw.ShapeMismatch):
        rnsw.rns_tile_conv(g, d, system, mts[:2])
    with pytest.raises(rnsw.ShapeMismatch):
        rnsw.rns_tile_conv(g, d, system, mts[::-1])
    small = rnsw.RnsSystem((7, 11, 13))
    with pytest.raises(rnsw.DynamicRangeExceeded):
        rnsw.rns_tile_conv(g, d, small, rnsw.reduce_for_system(rnsw.cached_transforms(2, 3), small))
    with pytest.raises(rnsw.ShapeMismatch):
        rnsw.rns_tile_conv(g, np.zeros((5, 5), np.int8), system, mts)
