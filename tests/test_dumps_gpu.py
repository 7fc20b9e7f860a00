"""The BASELINE dump pipelines, pinned at every dump point against the
reference itself (tests/golden/golden_dumps.json, made by
tests/golden/make_golden_dumps.py from oracle/_ref = proj/core built from
source):

* cfg3 — cylinder 8192 x 4096, FHP-III, p = 0.01: coarse_grain(32) every 100
  steps up to 5,000, through the asynchronous dump pipeline (cells_async
  enqueued behind the step kernels, collected with cells_wait);
* cfg2 — channel 4096 x 2048, FHP-III, p = 0.01: coarse_grain(16) and
  velocity_profile every 1,000 steps up to 10,000.

The cell doubles (rho, ux, uy: observables.cpp:49-82) and the profile
(observables.cpp:84-102) must equal the reference's bit for bit, the state
digest (lattice.cpp:122-132) and the forcing swaps too.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1208_2428_b200 as P
from paper_1208_2428_b200.observables import finalize_cells, finalize_profile

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_dumps.json")


def _cells_hash(f):
    h = hashlib.sha256()
    for a, t in ((f.nodes, np.int32), (f.particles, np.int32), (f.rho, np.float64),
                 (f.ux, np.float64), (f.uy, np.float64)):
        h.update(np.ascontiguousarray(a, t).tobytes())
    return h.hexdigest()


def _profile_hash(mean_ux, count):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(mean_ux, np.float64).tobytes())
    h.update(np.ascontiguousarray(count, np.int32).tobytes())
    return h.hexdigest()


def _configs():
    if not os.path.exists(GOLDEN):
        return []
    return json.load(open(GOLDEN))["configs"]


@pytest.mark.parametrize("c", _configs(), ids=lambda c: c["name"])
def test_dump_points_equal_reference(c, port, tables):
    mask = port.cylinder(c["W"], c["H"]) if c.get("geometry") == "cylinder" else None
    e = P.Engine(c["W"], c["H"])
    e.set_table(tables[c["table"]])
    if mask is not None:
        e.set_obstacles(mask)
    e.init(c["seed"], c["density"])
    e.swaps(reset=True)
    every, block = c["every"], c["block"]
    for d in c["dumps"]:
        s0 = d["step"] - every
        e.advance_async(c["seed"], P.bernoulli_threshold(c["force_p"]), s0, every)
        e.cells_async(block)  # the dump pipeline: sums enqueued behind the steps
        field = finalize_cells(block, *e.cells_wait())
        assert _cells_hash(field) == d["cells"], (c["name"], d["step"])
        if c.get("profile"):
            _, mean, cnt = finalize_profile(*e.rows())
            assert _profile_hash(mean, cnt) == d["profile"], (c["name"], d["step"])
        assert list(e.observables()) == d["obs"], (c["name"], d["step"])
        assert e.swaps() == d["swaps"], (c["name"], d["step"])
        assert P.state_digest(e.download()) == d["digest"], (c["name"], d["step"])
