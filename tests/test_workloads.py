"""Seeded workload generation: deterministic, byte-identical to the golden
digests, with the value distributions BASELINE.json states."""
import numpy as np

from paper_2007_12216_b200 import workloads as W
from golden_util import digests, sha


def test_config1_inputs_match_golden_digest():
    case, w, x = W.config1()
    d = digests()["cfg1"]
    assert sha(x) == d["x"] and sha(w) == d["w"]
    assert x.min() >= -32 and x.max() <= 31 and w.min() >= -32 and w.max() <= 31
    assert case.declared_bound == 589_824


def test_config3_inputs_match_golden_digest():
    case, w, x = W.config3()
    d = digests()["cfg3"]
    assert sha(x) == d["x"] and sha(w) == d["w"]
    assert x.min() >= -16 and x.max() <= 15 and case.declared_bound == 819_200


def test_config5_cases_and_inputs():
    w, x = W.config5_operands()
    d = digests()["cfg5/direct"]
    assert sha(x) == d["x"] and sha(w) == d["w"]
    assert x.min() >= 0 and x.max() <= 127 and np.abs(w.astype(int)).max() <= 127
    names = [c.name for c in W.config5_cases()]
    assert len(names) == 13
    assert "cfg5-F12-253x251x247" not in names and "cfg5-F10-253x251x247" in names
    for c in W.config5_cases():
        assert c.declared_bound <= 7_228_674


def test_vgg_inputs_match_golden_digests():
    ws = W.vgg16_weights()
    dg = digests()
    for (name, *_), w in zip(W.VGG16_LAYERS, ws):
        assert sha(w) == dg[f"vgg16/{name}"]["w"]
    assert sha(W.vgg16_images(1)) == dg["vgg16/image0"]["x"]
    shard = W.vgg16_images(2, start=1)
    assert np.array_equal(shard[0], W.vgg16_images(1, start=1)[0])
    bounds = W.vgg16_bounds(ws)
    assert bounds == [dg[f"vgg16/{n}"]["bound"] for n, *_ in W.VGG16_LAYERS]


def test_vgg_streams_are_independent():
    """make_rng keeps only the first 8 bytes of a string label (the
    reference's rw/cli.py:82-94 fold), so per-image / per-layer indices travel
    as separate entropy words: every image and every layer is its own draw."""
    imgs = W.vgg16_images(4, start=30)
    for i in range(4):
        for j in range(i + 1, 4):
            assert (imgs[i] != imgs[j]).mean() > 0.9
    ws = W.vgg16_weights()
    same_shape = [i for i, (_, _, c, k, _) in enumerate(W.VGG16_LAYERS) if (c, k) == (512, 512)]
    assert len(same_shape) == 5
    for i in same_shape[1:]:
        assert (ws[i] != ws[same_shape[0]]).mean() > 0.9
    # the fold itself, as the reference has it
    assert W.make_rng(1, "vgg16/image/1").integers(0, 1 << 30) == W.make_rng(1, "vgg16/im").integers(0, 1 << 30)


def test_vgg_direct_ops():
    assert W.VGGConfig(batch=1).direct_ops() == sum(
        2 * s * s * c * k * 9 for _, s, c, k, _ in W.VGG16_LAYERS)
    assert abs(W.VGGConfig(batch=1).direct_ops() / 1e9 - 30.7) < 0.1
