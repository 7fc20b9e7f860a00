"""The drop-in at the reference's own symbol: proj/core built from its own
sources with integration/backend_cuda.patch (Backend::Cuda in fhp::advance,
step.cpp:103-133) and the shim integration/cuda_backend.cpp, linked against
libfhpg.so (integration/Makefile -> oracle/_ref/dropin/dropin_check).
dropin_check runs the reference's acceptance criterion 3 generator (24
configs, acceptance.cpp:58-97) Scalar vs Cuda, the all-backends case
(test_backends.cpp:161-171) with Cuda added, and the bit-plane path (FHP-III
from data/fhp3.fhptab, Strips vs Cuda vs Cuda over 2 strips)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin", "dropin_check")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in build absent (needs the reference tree)")
def test_reference_runs_backend_cuda_bit_exact():
    r = subprocess.run([BIN, "check", os.path.join(ROOT, "data", "fhp3.fhptab")],
                       capture_output=True, text=True, timeout=900)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert r.returncode == 0, r.stdout + r.stderr
    assert lines[0]["mismatches"] == 0
    assert lines[1]["agree"] and lines[2]["agree"]
    assert lines[-1]["failures"] == 0
