"""CPU checks of the committed full-size oracle digests (tests/golden/fullsize_*.json,
written by tools/oracle_golden.py from oracle/ + synth/ only): they exist for all five
BASELINE configs, were computed on the current synthetic inputs (input SHA-256), and
cover every subset.  The GPU comparison is tests/test_gpu_fullsize.py."""
import json
import os

from synth import build_config
from _digest import input_sha

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return json.load(open(os.path.join(GOLDEN, f"fullsize_{name}.json")))


def test_golden_digests_cover_every_config():
    """the committed digests exist for all five BASELINE configs and match the current inputs
    (the comparison itself is tests/test_gpu_fullsize.py)."""
    for name in ("C1", "C2", "C3", "C4", "C5"):
        gold = golden(name)
        h = build_config(name)
        assert gold["input_sha256"] == input_sha(h)
        assert [w["T"] for w in gold["ands"]] == [list(T) for T in h.subsets]
        assert len(gold["layers"]) == len(h.layers)
        assert all("or_edges" in w and "cc1_ranked" in w and "gt_topk" in w for w in gold["ands"])


