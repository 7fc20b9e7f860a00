"""The BASELINE configs at their full step counts against the reference's
own results (tests/golden/golden_long.json, made by
tests/golden/make_golden_long.py with the unmodified reference library):
cfg2 (4096x2048 channel, forcing, 10,000 steps), cfg3 (8192x4096 cylinder,
forcing, 5,000 steps), cfg4 (16384^2, 20 steps). Bit-exact digest, accepted
forcing swaps, mass and momentum; the runs are chunked the way a dump
cadence would split them (state resident on the device between calls)."""
import json
import os

import pytest

import paper_1208_2428_b200 as P

pytestmark = pytest.mark.gpu

LONG = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_long.json")


def _configs():
    if not os.path.exists(LONG):
        return []
    return json.load(open(LONG))["configs"]


@pytest.mark.parametrize("c", _configs(), ids=lambda c: c["name"])
def test_baseline_config_full_length(c, tables, port):
    e = P.Engine(c["W"], c["H"])
    e.set_table(tables[c["table"]])
    if c.get("geometry") == "cylinder":
        e.set_obstacles(port.cylinder(c["W"], c["H"]))
    e.init(c["seed"], c["density"])
    chunk = 1000 if c["steps"] >= 1000 else c["steps"]
    swaps, s = 0, 0
    while s < c["steps"]:
        n = min(chunk, c["steps"] - s)
        swaps += e.advance(c["seed"], c["force_p"], s, n)
        s += n
    assert port.digest(e.download()) == c["digest"]
    assert swaps == c["swaps"]
    assert list(e.observables()) == c["obs"]
    e.close()
