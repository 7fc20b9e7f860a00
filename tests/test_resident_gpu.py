"""The shared-memory-resident kernel for small bit-plane lattices
(fhpg_step_resident.cu): a whole multi-step advance call in one cooperative
launch, time-blocked with deep halos (halo rows recomputed by neighbouring
CTAs). Bit-exact against the oracle and against the streaming kernels
(fhpg_select_path 3) on adversarial states: both row parities at CTA row
boundaries, step counts that are not multiples of the halo depth, forcing,
every rule with a circuit, walls and obstacles, nonzero first steps. (cfg1 itself, FHP-I 1024^2 for 1000 steps against the
reference's digest, is tests/test_parity_gpu.py::test_cfg1_fhp1_1024, which
now runs on this kernel.)"""
import pytest

import paper_1208_2428_b200 as P

pytestmark = pytest.mark.gpu


def _engine(W, H, table, mask, state, path="auto"):
    e = P.Engine(W, H)
    e.set_table(table)
    if path != "auto":
        e.select_path(path)
    e.set_obstacles(mask)
    e.upload(state)
    return e


@pytest.mark.parametrize("W,H", [(1024, 1024), (1024, 3), (1024, 37), (2048, 301), (4096, 150),
                                 (1024, 2000)])
@pytest.mark.parametrize("rule,fp", [("fhp3", 0.0), ("fhp3", 0.3), ("fhp1", 0.0), ("default", 0.05)])
def test_resident_equals_oracle_and_streaming(W, H, rule, fp, port, tables):
    state, mask = port.scramble(W, H, W + 7 * H)
    t = tables[rule]
    a = _engine(W, H, t, mask, state)
    b = _engine(W, H, t, mask, state, "streaming")
    n0 = a.step_launches
    resident = a.resident_depth(fp) > 0
    assert b.resident_depth(fp) == 0
    if W * H <= 1 << 20 and not fp:
        assert resident                   # the small no-forcing shapes always fit
    swa = a.advance(9, fp, 13, 11)       # 11 steps: not a multiple of the halo depth
    # one launch for the whole call (else one step kernel per step + the column keys)
    assert a.step_launches - n0 == (1 if resident else 12)
    swb = b.advance(9, fp, 13, 11)
    assert swa == swb
    out = a.download()
    assert (out == b.download()).all()
    if W * H <= 1 << 20:
        ref, rsw = port.advance(state, t, 9, port.threshold(fp), 13, 11, mask=mask)
        assert (out == ref).all()
        assert swa == rsw
    # a second call continues exactly (buffer parity after the flips)
    assert a.advance(9, fp, 24, 6) == b.advance(9, fp, 24, 6)
    assert (a.download() == b.download()).all()


@pytest.mark.parametrize("W,H", [(2048, 301), (4096, 150), (1024, 1024)])
def test_mixed_single_and_multi_step_calls(W, H, port, tables):
    """Single-step calls run the streaming kernels (the ring kernel keeps no
    periodic-wrap sectors in the plane rows), multi-step calls the resident
    kernel (which rebuilds the wrap words from the data): any interleaving
    equals the oracle."""
    state, mask = port.scramble(W, H, 3 * W + H)
    t = tables["fhp3"]
    a = _engine(W, H, t, mask, state)
    step, sw = 40, 0
    for n in (1, 5, 1, 1, 7, 1):
        sw += a.advance(2, 0.0, step, n)
        step += n
    if W * H <= 1 << 20:
        ref, rsw = port.advance(state, t, 2, 0, 40, step - 40, mask=mask)
        assert (a.download() == ref).all()
        assert sw == rsw
    else:
        b = _engine(W, H, t, mask, state, "streaming")
        b.advance(2, 0.0, 40, step - 40)
        assert (a.download() == b.download()).all()


def test_resident_plan_crossover(tables):
    """The resident kernel takes unforced lattices up to 4M sites and forced
    ones up to 2M (measured crossovers, fhpg_step_resident.cu): 2048^2 runs
    resident unforced and streaming forced; 2048 x 1024 resident either way."""
    big = P.Engine(2048, 2048)
    big.set_table(tables["fhp3"])  # a circuit rule: the bit-plane layout
    assert big.resident_depth(0.0) > 0 and big.resident_depth(0.01) == 0
    half = P.Engine(2048, 1024)
    half.set_table(tables["fhp3"])
    assert half.resident_depth(0.0) > 0 and half.resident_depth(0.01) > 0
    big.close()
    half.close()
