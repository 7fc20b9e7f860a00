"""Shared fixtures. `gpu`-marked tests need a CUDA device (run on the B200 box);
everything else runs on CPU. The oracle (oracle/) is the checker only."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def tables(golden):
    return {k: np.frombuffer(bytes.fromhex(v), np.uint8).copy() for k, v in golden["tables"].items()}


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()
