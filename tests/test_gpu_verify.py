"""The reference's acceptance sweep C3 (t/test_acceptance.py:126-144, 217
randomized layers over 12 tile shapes incl. F(14x14,5x5), 3 RNS systems) on
the GPU: every output must equal the reference's own layer_conv output,
whose SHA-256 digests are frozen in tests/golden/verify.json."""
import json

import numpy as np
import pytest

from golden_util import GOLDEN, sha

pytestmark = pytest.mark.gpu


def test_reference_verify_sweep_bit_exact():
    import paper_2007_12216_b200 as rnsw
    from paper_2007_12216_b200 import workloads as W

    gold = json.loads((GOLDEN / "verify.json").read_text())
    cases = W.verify_cases(2020)
    assert len(cases) == len(gold) == 217
    failures = []
    for case, ref in zip(cases, gold):
        w, x = W.verify_operands(case)
        spec = rnsw.LayerSpec(h=case["h"], w=case["w"], c=case["c"], k=case["k"], r=case["r"],
                              padding=case["pad"], batch=case["batch"], tile_m=case["tile_m"])
        y = rnsw.layer_conv(spec, w, x, rnsw.RnsSystem(case["moduli"]))
        if sha(y) != ref["y"]:
            failures.append(ref["label"])
    assert not failures, failures[:5]
