"""CPU checks of the C ABI boundary: libfhpg.so loads and exports every symbol
include/*.h declares; host-only entry points behave like the reference; the
engine refuses to run without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1208_2428_b200 as P
from paper_1208_2428_b200 import engine as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if h.endswith(".h"):
            src = open(os.path.join(ROOT, "include", h)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(fhpg_\w+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    lib = P.load_library()
    syms = declared_symbols()
    assert len(syms) >= 20
    for name in sorted(syms):
        assert hasattr(lib, name), name
    # the Python binding covers every declared entry point
    assert syms == set(E.SIGNATURES), syms ^ set(E.SIGNATURES)


def test_bernoulli_threshold_matches_reference_expression(port):
    for p in (0.0, 1e-9, 0.01, 0.3, 0.5, 0.999999, 1.0, 2.0):
        assert P.bernoulli_threshold(p) == port.threshold(p)


def test_tables_match_golden_and_validate(tables):
    for v in ("default", "fhp1", "fhp3"):
        t = P.build_table(v)
        assert (t == tables[v]).all(), v
        assert P.validate_table(t) == 0


def test_fhp3_is_collision_saturated_and_symmetric(tables):
    t = tables["fhp3"]
    changed = sum(1 for s in range(128) if t[s] != s or t[256 + s] != s)
    assert changed == 76  # FHP-III: 76 colliding fluid states

    def rot(s, k):
        m = s & 0x3F
        return (s & 0xC0) | (((m << k) | (m >> (6 - k))) & 0x3F)

    for ch in (0, 1):
        for s in range(256):
            assert t[ch * 256 + rot(s, 1)] == rot(t[ch * 256 + s], 1)
    perm = [4, 3, 2, 1, 0, 5]  # mirror y -> -y: NW<->SW, NE<->SE

    def mir(s):
        o = s & 0xC0
        for k in range(6):
            if s >> k & 1:
                o |= 1 << perm[k]
        return o

    for s in range(128):
        assert t[256 + mir(s)] == mir(t[s])
    # each chirality slice permutes the fluid states (survey Appendix B)
    for ch in (0, 1):
        assert sorted(t[ch * 256: ch * 256 + 128].tolist()) == list(range(128))


def test_fhp1_has_no_rest_rules(tables):
    t = tables["fhp1"]
    for s in range(64, 128):
        assert t[s] == s and t[256 + s] == s
    assert t[0b00001001] == 0b00100100 and t[256 + 0b00001001] == 0b00010010
    assert t[0b00010101] == 0b00101010


def test_unknown_variant_rejected():
    with pytest.raises(ValueError):
        P.build_table("fhp9")


def test_validator_flags_corruption(tables):
    t = tables["default"].copy()
    t[1] = 0
    assert P.validate_table(t) > 0


def test_engine_fails_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present: covered by the gpu tests")
    except ImportError:
        pass
    with pytest.raises(P.FhpgError):
        P.Engine(64, 34)
