"""Checkpoint / resume: the FHPCKPT1 format and exact
resumption of a device-resident run."""
import numpy as np
import pytest

import paper_1208_2428_b200 as P
from paper_1208_2428_b200 import checkpoint as K


def test_state_digest_matches_oracle_digest(port):
    for (W, H, seed) in ((48, 33, 1), (100, 9, 2), (513, 17, 3)):
        s, _ = port.scramble(W, H, seed)
        assert P.state_digest(s) == port.digest(s)
    assert P.state_digest(np.zeros(0, np.uint8)) == 0xCBF29CE484222325


def test_format_round_trip_and_corruption(tmp_path, port, tables):
    s, _ = port.scramble(64, 20, 7)
    ck = K.Checkpoint(64, 20, 123, 2**63 + 5, 0.01, 42, tables["fhp3"], s)
    path = str(tmp_path / "a.ck")
    K.save(path, ck)
    raw = open(path, "rb").read()
    assert len(raw) == K.HEADER_BYTES + 64 * 20 and raw[:8] == b"FHPCKPT1"
    back = K.load(path)
    assert (back.width, back.height, back.next_step, back.seed, back.force_p, back.swaps) == \
        (64, 20, 123, 2**63 + 5, 0.01, 42)
    assert (back.table == tables["fhp3"]).all() and (back.state == s).all()
    bad = bytearray(raw)
    bad[K.HEADER_BYTES + 5] ^= 0x10
    with pytest.raises(RuntimeError, match="digest"):
        K.parse(bytes(bad))
    with pytest.raises(RuntimeError, match="magic"):
        K.parse(b"FHPTAB01" + raw[8:])
    with pytest.raises(RuntimeError, match="size"):
        K.parse(raw[:-1])


@pytest.mark.gpu
def test_resume_equals_uninterrupted(tmp_path, port, tables):
    W, H, seed, fp = 1056, 70, 99, 0.05
    s, m = port.scramble(W, H, seed)

    def fresh():
        e = P.Engine(W, H)
        e.set_table(tables["fhp3"])
        e.set_obstacles(m)
        e.upload(s)
        return e

    e = fresh()
    total = e.advance(seed, fp, 0, 30)
    want = e.download()
    e1 = fresh()
    sw = e1.advance(seed, fp, 0, 12)
    path = str(tmp_path / "r.ck")
    K.save(path, K.capture(e1, 12, seed, fp, sw, tables["fhp3"]))
    ck = K.load(path)
    e2 = P.Engine(W, H)
    K.restore(e2, ck)
    sw2 = e2.advance(ck.seed, ck.force_p, ck.next_step, 30 - ck.next_step)
    assert (e2.download() == want).all()
    assert ck.swaps + sw2 == total
