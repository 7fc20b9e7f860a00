"""Parity of the bit-plane step path (csrc/fhpg_step_planes.cu) with the
oracle and with the byte paths.

The engine picks the bit-plane layout automatically for the FHP-III table
when W % 1024 == 0; these tests pin every entry point that crosses the
layout boundary (upload / init / obstacles / download / observables / table
and path switches / row strips / split steps) and the kernel itself on
adversarial states (particles on walls and obstacles, bit 7 that disagrees
with the mask, nonzero first_step, forcing up to p = 1). Bit-exact.
"""
import numpy as np
import pytest

import paper_1208_2428_b200 as P

pytestmark = pytest.mark.gpu


def engine(W, H, table, mask=None, state=None, path="auto"):
    e = P.Engine(W, H)
    e.select_path(path)
    e.set_table(table)
    if mask is not None:
        e.set_obstacles(mask)
    if state is not None:
        e.upload(state)
    return e


def test_path_selection(tables):
    assert engine(1024, 8, tables["fhp3"]).path == "planes"
    assert engine(16384, 8, tables["fhp3"]).path == "planes"
    assert engine(1024, 8, tables["default"]).path == "planes"  # the reference's rule as a circuit
    assert engine(1024, 8, tables["fhp1"]).path == "planes"
    t = tables["fhp3"].copy()
    t[3], t[5] = t[5], t[3]  # any other table: byte LUT path
    assert engine(1024, 8, t).path == "bytes"
    assert engine(1056, 8, tables["fhp3"]).path == "bytes"
    assert engine(1024, 8, tables["fhp3"], path="bytes").path == "bytes"
    assert engine(1024, 8, tables["fhp3"], path="generic").path == "generic"
    e = engine(2048, 8, tables["fhp3"])
    e.force_generic(True)
    assert e.path == "generic"
    e.force_generic(False)
    assert e.path == "planes"


@pytest.mark.parametrize("case", range(24))
def test_planes_against_oracle(case, port, tables):
    rng = np.random.default_rng(7000 + case)
    W = int(rng.choice([1024, 2048, 3072, 4096, 5120]))
    H = int(rng.choice([3, 4, 5, 6, 37, 64, 131]))
    fp = float(rng.choice([0.0, 0.0, 0.01, 0.3, 1.0]))
    seed = int(rng.integers(0, 2**63))
    steps = int(rng.integers(1, 13))
    first = int(rng.integers(0, 10**6))
    s, m = port.scramble(W, H, seed)
    ref, rsw = port.advance(s, tables["fhp3"], seed, port.threshold(fp), first, steps, mask=m)
    e = engine(W, H, tables["fhp3"], m, s)
    assert e.path == "planes"
    sw = e.advance(seed, fp, first, steps)
    out = e.download()
    assert (out == ref).all(), (W, H, fp, steps, np.argwhere(out != ref)[:5])
    assert sw == rsw


@pytest.mark.parametrize("fp", [0.0, 0.01])
def test_planes_equal_byte_path_wide(fp, port, tables):
    W, H = 16384, 301
    s, m = port.scramble(W, H, 99)
    a = engine(W, H, tables["fhp3"], m, s)
    b = engine(W, H, tables["fhp3"], m, s, path="bytes")
    assert a.path == "planes" and b.path == "bytes"
    swa = a.advance(5, fp, 1000, 17)
    swb = b.advance(5, fp, 1000, 17)
    assert (a.download() == b.download()).all()
    assert swa == swb
    ref, rsw = port.advance(s, tables["fhp3"], 5, port.threshold(fp), 1000, 17, mask=m)
    assert (a.download() == ref).all() and swa == rsw


def test_step_count_zero_keeps_uploaded_bytes_planes(port, tables):
    s, m = port.scramble(1024, 20, 5)
    s[3, 7] |= 0x80  # bit 7 without an obstacle
    s[4, 9] &= 0x7F  # obstacle without bit 7
    m[4, 9] = 1
    e = engine(1024, 20, tables["fhp3"], m, s)
    assert e.path == "planes"
    assert e.advance(1, 0.5, 10, 0) == 0
    assert (e.download() == s).all()
    assert e.observables() == port.global_obs(s)
    # the first step derives bit 7 from the mask, like the reference
    ref, rsw = port.advance(s, tables["fhp3"], 1, port.threshold(0.5), 10, 3, mask=m)
    assert e.advance(1, 0.5, 10, 3) == rsw
    assert (e.download() == ref).all()


def test_layout_switches_mid_run(port, tables):
    W, H = 2048, 70
    s, m = port.scramble(W, H, 8)
    e = engine(W, H, tables["fhp3"], m, s)
    ref = s
    custom = tables["fhp3"].copy()
    custom[3], custom[5] = custom[5], custom[3]  # no circuit: byte LUT path
    tabs = dict(tables, custom=custom)
    plan = [("fhp3", 4), ("default", 3), ("custom", 3), ("fhp3", 5), ("fhp1", 2), ("custom", 2),
            ("fhp3", 6)]
    step = 100
    for name, n in plan:
        e.set_table(tabs[name])
        assert e.path == ("bytes" if name == "custom" else "planes")
        sw = e.advance(3, 0.2, step, n)
        ref, rsw = port.advance(ref, tabs[name], 3, port.threshold(0.2), step, n, mask=m)
        assert (e.download() == ref).all(), name
        assert sw == rsw
        step += n
    # path switches keep the state too
    for path in ("bytes", "generic", "auto"):
        e.select_path(path)
        sw = e.advance(3, 0.2, step, 3)
        ref, rsw = port.advance(ref, tables["fhp3"], 3, port.threshold(0.2), step, 3, mask=m)
        assert (e.download() == ref).all(), path
        step += 3


def test_obstacles_and_init_in_planes_mode(port, tables):
    W, H = 4096, 90
    cyl = port.cylinder(W, H)
    e = engine(W, H, tables["fhp3"])
    e.set_obstacles(cyl)
    e.init(12, 0.3)
    ref = port.init(W, H, 12, 0.3, mask=cyl)
    assert (e.download() == ref).all()
    cyl = cyl.copy()
    cyl[0] = cyl[-1] = 1  # init_impl makes the wall rows obstacles (lattice.cpp:80-84)
    e.advance(12, 0.05, 0, 7)
    ref, _ = port.advance(ref, tables["fhp3"], 12, port.threshold(0.05), 0, 7, mask=cyl)
    assert (e.download() == ref).all()
    # new obstacles mid-run: bit 7 follows the mask at once (lattice.cpp:25-29)
    m2 = np.zeros((H, W), np.uint8)
    m2[20:30, 100:200] = 1
    e.set_obstacles(m2)
    ref = (ref & 0x7F) | (m2 << 7)
    assert (e.download() == ref).all()
    e.advance(12, 0.05, 7, 5)
    ref, _ = port.advance(ref, tables["fhp3"], 12, port.threshold(0.05), 7, 5, mask=m2)
    assert (e.download() == ref).all()


def test_observables_in_planes_mode(port, tables):
    W, H = 3072, 77
    s, m = port.scramble(W, H, 31)
    e = engine(W, H, tables["fhp3"], m, s)
    e.advance(2, 0.1, 0, 9)
    ref, _ = port.advance(s, tables["fhp3"], 2, port.threshold(0.1), 0, 9, mask=m)
    assert e.observables() == port.global_obs(ref)
    for B in (1, 4, 16, 33):
        for g, x in zip(e.cells(B), port.cells(ref, B)):
            assert (g == x).all(), B
    px, fl = e.rows()
    epx, efl = port.rows(ref)
    assert (px == epx).all() and (fl == efl).all()
    # observing does not disturb the resident state
    e.advance(2, 0.1, 9, 4)
    ref, _ = port.advance(ref, tables["fhp3"], 2, port.threshold(0.1), 9, 4, mask=m)
    assert (e.download() == ref).all()


def test_split_steps_planes(port, tables):
    for (W, H) in ((1024, 40), (2048, 3), (2048, 4), (16384, 37)):
        s, m = port.scramble(W, H, 21)
        b = engine(W, H, tables["fhp3"], m, s)
        assert b.path == "planes"
        thr = P.bernoulli_threshold(0.2)
        b.swaps(reset=True)
        for step in range(30, 36):
            b.advance_part(7, thr, step, 0)
            b.advance_part(7, thr, step, 1)
        ref, rsw = port.advance(s, tables["fhp3"], 7, thr, 30, 6, mask=m)
        assert (b.download() == ref).all(), (W, H)
        assert b.swaps() == rsw


@pytest.mark.parametrize("n", [2, 3, 5])
def test_local_strips_planes(n, port, tables):
    from paper_1208_2428_b200.strips import LocalStrips
    W, H = 2048, 67  # odd strip offsets: both row parities at strip starts
    s, m = port.scramble(W, H, 40 + n)
    ls = LocalStrips(W, H, n)
    ls.set_table(tables["fhp3"])
    assert all(e.path == "planes" for e in ls.engines)
    ls.set_obstacles(m)
    ls.upload(s)
    sw = ls.advance(11, 0.3, 2, 9)
    ref, rsw = port.advance(s, tables["fhp3"], 11, port.threshold(0.3), 2, 9, mask=m)
    assert (ls.download() == ref).all() and sw == rsw


def test_mass_conserved_full_size_planes(tables):
    W = H = 16384
    e = engine(W, H, tables["fhp3"])
    e.init(4, 0.2)
    assert e.path == "planes"
    m0, _, _ = e.observables()
    for k in range(3):
        e.advance(4, 0.0, 20 * k, 20)
        assert e.observables()[0] == m0


# --- precomputed-column chirality keys (ring kernel, chir_column / chir_bit) --
_M64 = (1 << 64) - 1
_GAMMA, _C1, _C2 = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def _mix64_np(z):
    z = z + np.uint64(_GAMMA)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_C1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_C2)
    return z ^ (z >> np.uint64(31))


def _carry_steps(seed, W, H, want, limit=200000, block=1 << 32):
    """Steps whose chirality column keys have a low word that carries for
    some row y in 1..H-1 but not for row 0 (lo32(K) > 2^32 - H), where
    key + y must carry into the high word (rng.hpp:25-33). With block =
    2^30: keys whose low word leaves its 2^30 block inside the rows (where
    the bit-plane kernels' folded column keys end and they re-key)."""
    base = int(_mix64_np(np.array([(seed + _GAMMA * 2) & _M64], np.uint64))[0])
    xs = np.arange(1, W + 1, dtype=np.uint64)
    found = []
    with np.errstate(over="ignore"):
        for s0 in range(0, limit, 4096):
            st = np.arange(s0, s0 + 4096, dtype=np.uint64)
            sk = _mix64_np(np.uint64(base) + st)
            keys = _mix64_np(sk[:, None] + xs[None, :]) + np.uint64(_GAMMA)
            lo = keys & np.uint64(block - 1)
            hit = np.argwhere(lo > np.uint64(block - H))
            for r, c in hit:
                found.append((int(st[r]), int(c)))
            if len({f[0] for f in found}) >= want:
                break
    steps = sorted({f[0] for f in found})[:want]
    return steps, found


def test_ring_carry_columns(port, tables):
    """Every site a chirality-dependent head-on pair (uniform 0x09), at steps
    where some column's low key word carries from some row on: the 64-bit
    key + row add must carry into the high word (chir_bit takes the sum)."""
    W, H, seed = 2048, 1000, 77
    steps, found = _carry_steps(seed, W, H, want=6)
    assert len(steps) >= 3
    s = np.full((H, W), 0x09, np.uint8)
    m = np.zeros((H, W), np.uint8)
    e = engine(W, H, tables["fhp3"], m, s)
    assert e.path == "planes"
    for st in steps:
        e.upload(s)
        e.advance(seed, 0.0, st, 1)
        ref, _ = port.advance(s, tables["fhp3"], seed, 0, st, 1, mask=m)
        out = e.download()
        assert (out == ref).all(), (st, [f for f in found if f[0] == st], np.argwhere(out != ref)[:5])



def test_ring_key_block_crossing(port, tables):
    """Steps where some column key's low word leaves its 2^30 block between
    two rows of the lattice: the ring kernel's folded column keys (ColKey,
    valid while lo + dy stays in the block) end there and the consumers
    re-key the band at that row (rekey_consumers)."""
    W, H, seed = 4096, 1000, 78
    steps, found = _carry_steps(seed, W, H, want=6, block=1 << 30)
    assert len(steps) >= 3
    s = np.full((H, W), 0x09, np.uint8)
    m = np.zeros((H, W), np.uint8)
    e = engine(W, H, tables["fhp3"], m, s)
    assert e.path == "planes"
    for st in steps:
        e.upload(s)
        e.advance(seed, 0.0, st, 1)
        ref, _ = port.advance(s, tables["fhp3"], seed, 0, st, 1, mask=m)
        out = e.download()
        assert (out == ref).all(), (st, [f for f in found if f[0] == st], np.argwhere(out != ref)[:5])


@pytest.mark.parametrize("W,H,fp,cap", [(16384, 1100, 0.3, 1), (16384, 1100, 0.0, 37),
                                        (4096, 131, 0.3, 0), (4096, 131, 1.0, 5),
                                        (3072, 64, 0.3, 0), (3072, 64, 0.0, 7),
                                        (1024, 64, 0.3, 3), (2048, 37, 0.01, 2)])
def test_key_span_cap(W, H, fp, cap, port, tables):
    """Column-key spans capped (fhpg_debug_key_span): the ring kernel re-keys
    every `cap` rows (cap 0 acts as 1), incl. across the extra CTAs' band
    switch; the per-warp kernel (W = 1024 x odd) hashes the rows past the
    cap from the step keys. Results are identical to the oracle."""
    s, m = port.scramble(W, H, W * 3 + H + cap)
    e = engine(W, H, tables["fhp3"], m, s, path="streaming")
    assert e.path == "planes"
    e.debug_key_span(cap)
    sw = e.advance(5, fp, 1234, 3)
    ref, rsw = port.advance(s, tables["fhp3"], 5, port.threshold(fp), 1234, 3, mask=m)
    out = e.download()
    assert (out == ref).all(), np.argwhere(out != ref)[:5]
    assert sw == rsw


@pytest.mark.parametrize("cap", [1, 7, 0xFFFFFFFF])
def test_key_span_cap_strips(cap, port, tables):
    """Re-keying inside the boundary-row launches of a multi-strip engine
    (interior rows and each strip's first / last row as a second row range
    of the ring kernel), with forcing; bit-exact with the oracle."""
    W, H = 4096, 300
    s, m = port.scramble(W, H, 4242 + (cap & 0xFF))
    e = P.Engine(W, H, strips=3, devices=[0, 0, 0])
    e.set_table(tables["fhp3"])
    e.set_obstacles(m)
    e.upload(s)
    e.debug_key_span(cap)
    sw = e.advance(9, 0.3, 501, 4)
    ref, rsw = port.advance(s, tables["fhp3"], 9, port.threshold(0.3), 501, 4, mask=m)
    out = e.download()
    assert (out == ref).all(), np.argwhere(out != ref)[:5]
    assert sw == rsw


@pytest.mark.parametrize("W,H,fp", [(16384, 1100, 0.0), (16384, 1100, 0.3), (12288, 1500, 0.05),
                                    (16384, 2000, 1.0)])
def test_ring_extra_ctas(W, H, fp, port, tables):
    """Widths whose band count leaves SMs over (8 bands x 18 segments = 144
    of 148 SMs at W = 16384; 6 x 24 at 12288): the spare CTAs take the last
    rows of two bands each, switching bands mid-kernel (key table rebuilt
    behind a consumer barrier, ring continuing across the switch)."""
    s, m = port.scramble(W, H, W + H)
    e = engine(W, H, tables["fhp3"], m, s)
    assert e.path == "planes"
    sw = e.advance(11, fp, 77, 3)
    ref, rsw = port.advance(s, tables["fhp3"], 11, port.threshold(fp), 77, 3, mask=m)
    out = e.download()
    assert (out == ref).all(), np.argwhere(out != ref)[:5]
    assert sw == rsw


@pytest.mark.parametrize("case", range(16))
@pytest.mark.parametrize("rule", ["default", "fhp1"])
def test_other_rules_planes_against_oracle(rule, case, port, tables):
    """The reference's own DEFAULT rule and FHP-I on the bit-plane path (their
    circuits, def_* / fhp1_*): adversarial states, obstacles, forcing up to
    p = 1, nonzero first_step, every kernel (W = 1024 per-warp, >= 4096
    ring, 16384 x 1100 ring with the extra-CTA split)."""
    rng = np.random.default_rng(9100 + case)
    if case == 15:
        W, H = 16384, 1100
    else:
        W = int(rng.choice([1024, 2048, 4096, 6144]))
        H = int(rng.choice([3, 5, 37, 64, 131]))
    fp = float(rng.choice([0.0, 0.0, 0.01, 0.3, 1.0]))
    seed = int(rng.integers(0, 2**63))
    steps = int(rng.integers(1, 9))
    first = int(rng.integers(0, 10**6))
    s, m = port.scramble(W, H, seed)
    ref, rsw = port.advance(s, tables[rule], seed, port.threshold(fp), first, steps, mask=m)
    e = engine(W, H, tables[rule], m, s)
    assert e.path == "planes"
    sw = e.advance(seed, fp, first, steps)
    out = e.download()
    assert (out == ref).all(), (W, H, fp, steps, np.argwhere(out != ref)[:5])
    assert sw == rsw
