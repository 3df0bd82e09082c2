"""Pins for the committed golden fixtures (tests/golden/*.json, written by
tests/golden/make_golden.py which calls only oracle.gf).

The fixtures are compared with values derived independently in SURVEY.md Sec. 8(c)
(SHA-256 of the u64-LE histograms, totals, ranges) and with the nested-loop oracle on
prefix boxes, so a wrong fixture cannot pass."""
import hashlib
import json
import os
import struct

import pytest

import oracle
from paper_2405_07989_b200 import workloads as W

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(HERE, name + ".json")) as f:
        return json.load(f)


def hsha(h):
    return hashlib.sha256(struct.pack("<%dQ" % len(h), *h)).hexdigest()


SURVEY_HIST_SHA = {
    "C1": "49612ed76a991a2968f06a110a34a88d99c02da67f60cddfba5dd936cf154fd1",
    "C2": "f42facb340c129e12519e6a18459ddc21e5203b307e78456b8f1f683e5a704e3",
    "C2L": "2ca42f377ddc1ad1e41fed67b2246c454a24da2ae7b4f0f2873f62c3179ca5a4",
    "C3": "732d09b032db36b6c536250ec753ddae1612ccfae0e19df8ccd8c028897bcdbd",
    "C5": "6885d3842dce884d6316e55e69273494eeedeffaed4c8eeef2a899b2421be420",
}
SURVEY_COUNT = {"C1": 465, "C2": 681152, "C2L": 824598466, "C2XL": 2597173872,
                "C3": 100032405189, "C5": 4055053706}


@pytest.mark.parametrize("name", sorted(SURVEY_HIST_SHA))
def test_fixture_hist_hash(name):
    doc = load(name)
    assert hsha(doc["hist"]) == SURVEY_HIST_SHA[name]
    assert sum(doc["hist"]) == doc["count"] == SURVEY_COUNT[name]


def test_c5_properties():
    h = load("C5")["hist"]
    assert len(h) == 20001
    assert h[20] == 1 and sum(h[:20]) == 0          # shortest: (0,0,0,0,20)
    assert sum(h[19995:]) == 119976
    assert sum(1 for v in h if v) == 19542


def test_c5_top_length_bruteforce():
    # independent: rows of length 20000 are exactly (a1, a2, 0, 0, 0), a1 + a2 = 20000
    h = load("C5")["hist"]
    assert h[20000] == 20001


def test_c2xl_count():
    assert load("C2XL")["count"] == 2597173872


@pytest.mark.parametrize("name,prefix", [("C3", (100, 50)), ("C3", (0, 0, 0, 30)), ("C5", (19000, 500)),
                                         ("C2L", (300, 200))])
def test_fixture_box_consistency(oracle_mod, name, prefix):
    """The oracle's box histogram never exceeds the fixture's global histogram."""
    inst = W.CONFIGS[name]
    r = oracle.run(inst.n, inst.gens, box=(prefix[:-1], prefix[-1], prefix[-1]),
                   hist_len=oracle.hist_len_for(inst.n, inst.gens))
    h = load(name)["hist"]
    assert all(a <= b for a, b in zip(r["hist"], h))
    assert r["count"] == sum(r["hist"])
