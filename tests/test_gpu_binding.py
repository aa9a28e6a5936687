"""The reference-side ctypes binding (integration/flashbias_ctypes_binding.py,
numpy + libcudart only) reproduces the reference's own golden outputs."""

import json
import os
import sys

import numpy as np
import pytest

from oracle import flashbias_oracle as orc

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "integration"))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))
CASES = [c for c in json.load(open(os.path.join(HERE, "golden", "manifest.json")))["cases"] if c["kind"] == "flashbias"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_ctypes_binding_matches_reference(case):
    from flashbias_ctypes_binding import flashbias_attention_b200
    a = {k: G[f"{case['name']}/{k}"] for k in case["inputs"]}
    want = G[f"{case['name']}/o"]
    got = flashbias_attention_b200(a["q"], a["k"], a["v"], a["fq"], a["fk"], mask=case["mask"])
    assert orc.rel_max_err(got, want) <= 1e-5
    got16 = flashbias_attention_b200(a["q"], a["k"], a["v"], a["fq"], a["fk"], mask=case["mask"], precision="bf16")
    assert orc.rel_max_err(got16, want) <= 2e-2 or orc.rel_max_err(
        got16, orc.flashbias_attention(*(np.asarray(x, np.float32).astype(np.float64) for x in
                                         (a["q"], a["k"], a["v"], a["fq"], a["fk"])), mask=case["mask"])) <= 2e-2
