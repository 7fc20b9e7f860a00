"""TEST INFRASTRUCTURE ONLY — ctypes front-ends for the two CPU checkers.

* ``Port``  — oracle/liboracle.so, the plain-C restatement (fhp_oracle.c).
* ``Ref``   — oracle/_ref/libfhpref.so, the UNMODIFIED reference library
  (/root/reference/proj/core/src/*.cpp) behind oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module. The product (paper_1208_2428_b200) never does.

All state buffers are numpy uint8 arrays of shape (H, W): the reference's
storage columns 1..W (no ghost columns), bit 7 included.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfhpref.so")

u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)

BACKENDS = {"scalar": 0, "lanes": 1, "strips": 2, "tiles": 3}


def _ptr(a, t=u8p):
    return None if a is None else a.ctypes.data_as(t)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def bernoulli_threshold(p: float) -> int:
    """rng.hpp:37-42 threshold, computed with the identical double expression."""
    return (1 << 32) if p >= 1.0 else int(np.uint64(np.float64(p) * np.float64(4294967296.0)))


class Port:
    """Plain-C restatement of the reference path (fhp_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.fo_mix64.restype = C.c_uint64
        L.fo_mix64.argtypes = [C.c_uint64]
        L.fo_node_random.restype = C.c_uint64
        L.fo_node_random.argtypes = [C.c_uint64] * 5
        L.fo_bernoulli_threshold.restype = C.c_uint64
        L.fo_bernoulli_threshold.argtypes = [C.c_double]
        L.fo_build_default_table.argtypes = [u8p]
        L.fo_validate_table.argtypes = [u8p]
        L.fo_init.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, u8p, u8p]
        L.fo_advance.restype = C.c_uint64
        L.fo_advance.argtypes = [C.c_int, C.c_int, u8p, u8p, u8p, C.c_uint64, C.c_uint64,
                                 C.c_int64, C.c_int64]
        L.fo_digest.restype = C.c_uint64
        L.fo_digest.argtypes = [C.c_int, C.c_int, u8p]
        L.fo_global.argtypes = [C.c_int, C.c_int, u8p, i64p, i64p, i64p]
        L.fo_cells.argtypes = [C.c_int, C.c_int, u8p, C.c_int, i32p, i32p, i64p, i64p]
        L.fo_rows.argtypes = [C.c_int, C.c_int, u8p, i64p, i32p]
        L.fo_scramble.argtypes = [C.c_int, C.c_int, C.c_uint64, u8p, u8p]
        L.fo_cylinder.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, u8p]
        L.fo_step_strip.restype = C.c_uint64
        L.fo_step_strip.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, u8p, u8p, u8p, C.c_uint64,
                                    C.c_uint64, C.c_uint64, u8p]

    def mix64(self, z):
        return self.lib.fo_mix64(z)

    def node_random(self, seed, purpose, step, x, y):
        return self.lib.fo_node_random(seed, purpose, step, x, y)

    def threshold(self, p):
        return self.lib.fo_bernoulli_threshold(p)

    def default_table(self):
        t = np.zeros(512, np.uint8)
        self.lib.fo_build_default_table(_ptr(t))
        return t

    def validate_table(self, t):
        return self.lib.fo_validate_table(_ptr(_u8(t)))

    def init(self, W, H, seed, density, mask=None):
        out = np.zeros((H, W), np.uint8)
        m = None if mask is None else _u8(mask)
        self.lib.fo_init(W, H, seed, density, _ptr(m), _ptr(out))
        return out

    def advance(self, state, table, seed, force_thr, first_step, step_count, mask=None):
        """Returns (new_state, swaps); `state` is not modified."""
        s = _u8(state).copy()
        H, W = s.shape
        m = None if mask is None else _u8(mask)
        swaps = self.lib.fo_advance(W, H, _ptr(s), _ptr(m), _ptr(_u8(table)), seed,
                                    force_thr, first_step, step_count)
        return s, swaps

    def digest(self, state):
        s = _u8(state)
        return self.lib.fo_digest(s.shape[1], s.shape[0], _ptr(s))

    def global_obs(self, state):
        s = _u8(state)
        m, px, py = C.c_int64(), C.c_int64(), C.c_int64()
        self.lib.fo_global(s.shape[1], s.shape[0], _ptr(s), C.byref(m), C.byref(px), C.byref(py))
        return m.value, px.value, py.value

    def cells(self, state, B):
        s = _u8(state)
        H, W = s.shape
        cx, cy = (W + B - 1) // B, (H - 2 + B - 1) // B
        nodes = np.zeros(cx * cy, np.int32)
        parts = np.zeros(cx * cy, np.int32)
        px = np.zeros(cx * cy, np.int64)
        py = np.zeros(cx * cy, np.int64)
        self.lib.fo_cells(W, H, _ptr(s), B, _ptr(nodes, i32p), _ptr(parts, i32p),
                          _ptr(px, i64p), _ptr(py, i64p))
        return (nodes.reshape(cy, cx), parts.reshape(cy, cx), px.reshape(cy, cx),
                py.reshape(cy, cx))

    def scramble(self, W, H, seed):
        """Adversarial (state, mask) pair; see fo_scramble."""
        s = np.zeros((H, W), np.uint8)
        m = np.zeros((H, W), np.uint8)
        self.lib.fo_scramble(W, H, seed, _ptr(s), _ptr(m))
        return s, m

    def cylinder(self, W, H, cx=None, cy=None, R=None):
        """BASELINE config 3 obstacle: disc at (W/4, H/2), radius H/16."""
        cx = W / 4 if cx is None else cx
        cy = H / 2 if cy is None else cy
        R = H / 16 if R is None else R
        m = np.zeros((H, W), np.uint8)
        self.lib.fo_cylinder(W, H, cx, cy, R, _ptr(m))
        return m

    def step_strip(self, H, row0, src_with_halos, mask, table, seed, thr, step):
        """One step of a row strip (fo_step_strip). src_with_halos: (nrows+2, W)."""
        src = _u8(src_with_halos)
        nrows, W = src.shape[0] - 2, src.shape[1]
        dst = np.zeros((nrows, W), np.uint8)
        sw = self.lib.fo_step_strip(W, H, row0, nrows, _ptr(src), _ptr(_u8(mask)), _ptr(_u8(table)),
                                    seed, thr, step, _ptr(dst))
        return dst, sw

    def rows(self, state):
        s = _u8(state)
        H, W = s.shape
        px = np.zeros(H - 2, np.int64)
        fl = np.zeros(H - 2, np.int32)
        self.lib.fo_rows(W, H, _ptr(s), _ptr(px, i64p), _ptr(fl, i32p))
        return px, fl


class RefError(RuntimeError):
    pass


class Ref:
    """The reference library itself (compiled from /root/reference sources)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_mix64.restype = C.c_uint64
        L.ref_mix64.argtypes = [C.c_uint64]
        L.ref_node_random.restype = C.c_uint64
        L.ref_node_random.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64]
        L.ref_bernoulli.argtypes = [C.c_uint64, C.c_double]
        L.ref_build_table.argtypes = [u8p]
        L.ref_validate_table.argtypes = [u8p]
        L.ref_init.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, u8p, u8p]
        L.ref_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64,
                              C.c_int, C.c_int, u8p, u8p, u8p, u64p, i64p, i64p, i64p, u64p]
        L.ref_advance.argtypes = [C.c_int, C.c_int, u8p, u8p, u8p, C.c_uint64, C.c_double,
                                  C.c_int, C.c_int, C.c_int, C.c_int, u64p]
        L.ref_observables.argtypes = [C.c_int, C.c_int, u8p, i64p, i64p, i64p, u64p]
        L.ref_coarse_grain.argtypes = [C.c_int, C.c_int, u8p, C.c_int, i32p, i32p, i32p, i32p,
                                       f64p, f64p, f64p]
        L.ref_velocity_profile.argtypes = [C.c_int, C.c_int, u8p, f64p, i32p]
        L.ref_bench.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                C.c_uint64, C.c_int, C.c_int, u8p, C.c_int, f64p, f64p, u64p]
        L.ref_bench_file.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                     C.c_uint64, C.c_int, C.c_int, C.c_char_p, C.c_int, f64p,
                                     f64p, u64p]

    def _check(self, rc):
        if rc != 0:
            raise RefError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def mix64(self, z):
        return self.lib.ref_mix64(z)

    def node_random(self, seed, purpose, step, x, y):
        return self.lib.ref_node_random(seed, purpose, step, x, y)

    def bernoulli(self, w, p):
        return bool(self.lib.ref_bernoulli(w, p))

    def default_table(self):
        t = np.zeros(512, np.uint8)
        self.lib.ref_build_table(_ptr(t))
        return t

    def validate_table(self, t):
        return self.lib.ref_validate_table(_ptr(_u8(t)))

    def init(self, W, H, seed, density, mask=None):
        out = np.zeros((H, W), np.uint8)
        m = None if mask is None else _u8(mask)
        self._check(self.lib.ref_init(W, H, seed, density, _ptr(m), _ptr(out)))
        return out

    def run(self, W, H, steps, density, force_p, seed, table=None, mask=None,
            backend="strips", threads=None):
        """fhp::run(cfg, table). Returns dict(state, swaps, mass, px, py, digest)."""
        if threads is None:
            threads = max(1, min(os.cpu_count() or 1, H - 2)) if backend in ("strips", "tiles") else 1
        out = np.zeros((H, W), np.uint8)
        sw, m, px, py, dg = C.c_uint64(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_uint64()
        t = None if table is None else _u8(table)
        mk = None if mask is None else _u8(mask)
        self._check(self.lib.ref_run(W, H, steps, density, force_p, seed, BACKENDS[backend],
                                     threads, _ptr(t), _ptr(mk), _ptr(out), C.byref(sw),
                                     C.byref(m), C.byref(px), C.byref(py), C.byref(dg)))
        return dict(state=out, swaps=sw.value, mass=m.value, px=px.value, py=py.value,
                    digest=dg.value)

    def advance(self, state, table, seed, force_p, first_step, step_count, mask=None,
                backend="scalar", threads=1):
        s = _u8(state).copy()
        H, W = s.shape
        sw = C.c_uint64()
        t = None if table is None else _u8(table)
        mk = None if mask is None else _u8(mask)
        self._check(self.lib.ref_advance(W, H, _ptr(s), _ptr(mk), _ptr(t), seed, force_p,
                                         first_step, step_count, BACKENDS[backend], threads,
                                         C.byref(sw)))
        return s, sw.value

    def observables(self, state):
        s = _u8(state)
        m, px, py, dg = C.c_int64(), C.c_int64(), C.c_int64(), C.c_uint64()
        self.lib.ref_observables(s.shape[1], s.shape[0], _ptr(s), C.byref(m), C.byref(px),
                                 C.byref(py), C.byref(dg))
        return dict(mass=m.value, px=px.value, py=py.value, digest=dg.value)

    def coarse_grain(self, state, block):
        s = _u8(state)
        H, W = s.shape
        cx, cy = C.c_int(), C.c_int()
        self._check(self.lib.ref_coarse_grain(W, H, _ptr(s), block, C.byref(cx), C.byref(cy),
                                              None, None, None, None, None))
        n = cx.value * cy.value
        nodes = np.zeros(n, np.int32)
        parts = np.zeros(n, np.int32)
        rho, ux, uy = np.zeros(n), np.zeros(n), np.zeros(n)
        self._check(self.lib.ref_coarse_grain(W, H, _ptr(s), block, C.byref(cx), C.byref(cy),
                                              _ptr(nodes, i32p), _ptr(parts, i32p),
                                              _ptr(rho, f64p), _ptr(ux, f64p), _ptr(uy, f64p)))
        shp = (cy.value, cx.value)
        return dict(nodes=nodes.reshape(shp), particles=parts.reshape(shp),
                    rho=rho.reshape(shp), ux=ux.reshape(shp), uy=uy.reshape(shp))

    def velocity_profile(self, state):
        s = _u8(state)
        H, W = s.shape
        mu = np.zeros(H - 2)
        cnt = np.zeros(H - 2, np.int32)
        self.lib.ref_velocity_profile(W, H, _ptr(s), _ptr(mu, f64p), _ptr(cnt, i32p))
        return mu, cnt

    def bench(self, W, H, steps, warmup, density, force_p, seed, table=None,
              backend="strips", threads=None, repeats=1):
        if threads is None:
            threads = max(1, min(os.cpu_count() or 1, H - 2)) if backend in ("strips", "tiles") else 1
        mups, secs, dg = C.c_double(), C.c_double(), C.c_uint64()
        t = None if table is None else _u8(table)
        self._check(self.lib.ref_bench(W, H, steps, warmup, density, force_p, seed,
                                       BACKENDS[backend], threads, _ptr(t), repeats,
                                       C.byref(mups), C.byref(secs), C.byref(dg)))
        return dict(mups=mups.value, wall_seconds=secs.value, digest=dg.value, threads=threads)


    def bench_file(self, W, H, steps, warmup, density, force_p, seed, table_file=None,
                   backend="strips", threads=None, repeats=1):
        """run_bench with cfg.table_file: the reference loads the FHPTAB01 file itself."""
        if threads is None:
            threads = max(1, min(os.cpu_count() or 1, H - 2)) if backend in ("strips", "tiles") else 1
        mups, secs, dg = C.c_double(), C.c_double(), C.c_uint64()
        path = None if table_file is None else os.fsencode(table_file)
        self._check(self.lib.ref_bench_file(W, H, steps, warmup, density, force_p, seed,
                                            BACKENDS[backend], threads, path, repeats,
                                            C.byref(mups), C.byref(secs), C.byref(dg)))
        return dict(mups=mups.value, wall_seconds=secs.value, digest=dg.value, threads=threads)


def load_ref_or_none():
    try:
        return Ref()
    except (FileNotFoundError, OSError):
        return None
