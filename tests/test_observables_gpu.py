"""Observables on the device against the oracle (observables.cpp:27-102):
total mass / momentum, coarse_grain's integer cell sums and
velocity_profile's row sums, read straight from the bit planes (no unpack)
or from bytes; whole-lattice and multi-strip engines (strips that cut cell
rows); the asynchronous coarse-grain request of the dump pipeline, which
must see the state at the point it was enqueued even when steps are
enqueued behind it."""
import numpy as np
import pytest

import paper_1208_2428_b200 as P

pytestmark = pytest.mark.gpu


def _engine(W, H, state, mask, table, strips=None):
    e = P.Engine(W, H) if strips is None else P.Engine(W, H, strips=strips, devices=[0] * strips)
    e.set_table(table)
    e.set_obstacles(mask)
    e.upload(state)
    return e


@pytest.mark.parametrize("W,H", [(2048, 67), (1024, 40), (3072, 9), (512, 33)])
@pytest.mark.parametrize("strips", [None, 3])
def test_observables_equal_oracle(W, H, strips, port, tables):
    state, mask = port.scramble(W, H, W + H)
    e = _engine(W, H, state, mask, tables["fhp3"], strips)
    # after stepping the state is normalised (bit 7 = mask): compare on it
    e.advance(7, 0.1, 0, 3)
    out = e.download()
    assert e.path == ("planes" if W % 1024 == 0 else "bytes")
    assert e.observables() == port.global_obs(out)
    for B in (1, 3, 4, 16, 31, 32, 33, 64, 100):
        got = e.cells(B)
        ref = port.cells(out, B)
        for k in range(4):
            assert (got[k] == ref[k]).all(), (B, k)
    px, fl = e.rows()
    rpx, rfl = port.rows(out)
    assert (px == rpx).all() and (fl == rfl).all()


@pytest.mark.parametrize("strips", [None, 2])
def test_async_cells_see_the_state_at_the_request(strips, port, tables):
    W, H = 4096, 130
    state, mask = port.scramble(W, H, 5)
    e = _engine(W, H, state, mask, tables["fhp3"], strips)
    e.advance(3, 0.05, 0, 10)
    snap = e.download()
    e.cells_async(16)
    e.advance_async(3, P.bernoulli_threshold(0.05), 10, 25)  # enqueued behind the request
    got = e.cells_wait()
    ref = port.cells(snap, 16)
    for k in range(4):
        assert (got[k] == ref[k]).all(), k
    # the steps behind it ran: the state moved on
    e.synchronize()
    ref2, _ = port.advance(state, tables["fhp3"], 3, port.threshold(0.05), 0, 35, mask=mask)
    assert (e.download() == ref2).all()
    with pytest.raises(P.FhpgInvalidArgument):
        e.cells_wait()  # nothing pending


def test_cfg3_cells_at_dump_points(port, tables):
    """cfg3 geometry (cylinder) at the dump cadence's shape: cell sums of
    the plane lattice == the oracle's on the downloaded bytes."""
    W, H = 8192, 4096
    mask = port.cylinder(W, H)
    e = P.Engine(W, H)
    e.set_table(tables["fhp3"])
    e.set_obstacles(mask)
    e.init(3, 0.2)
    for s in range(0, 300, 100):
        e.advance(3, 0.01, s, 100)
        e.cells_async(32)
        got = e.cells_wait()
        ref = port.cells(e.download(), 32)
        for k in range(4):
            assert (got[k] == ref[k]).all(), (s, k)
