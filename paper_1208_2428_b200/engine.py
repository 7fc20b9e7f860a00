"""Python binding of the C ABI in include/fhpg.h (libfhpg.so).

Mirrors the reference's evolution interface (proj/core/include/fhp/step.hpp,
lattice.hpp, observables.hpp) on a device-resident lattice:

    eng = Engine(W, H)                 # Lattice(W, H)            lattice.cpp:10-17
    eng.set_table(table512)            # CollisionTable           collision.hpp:17-23
    eng.set_obstacles(mask)            # Lattice::set_obstacle    lattice.cpp:19-30
    eng.init(seed, density)            # init_lattice(cfg)        lattice.cpp:57-101
    swaps = eng.advance(seed, p, first_step, step_count)   # fhp::advance step.cpp:103-133
    eng.download()                     # Lattice::src() interior
    eng.observables()                  # total_mass/total_momentum observables.cpp:27-47

There is no CPU fallback: if libfhpg.so is missing or no CUDA device is
present, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FHPG_LIB overrides the engine library (A/B builds of kernel variants).
LIB_PATH = os.environ.get("FHPG_LIB") or os.path.join(_HERE, "lib", "libfhpg.so")

EINVAL = 2
ERUNTIME = 3

u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
vpp = C.POINTER(C.c_void_p)

# Every symbol include/fhpg.h declares, with (restype, argtypes).
SIGNATURES = {
    "fhpg_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "fhpg_create_strip": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(C.c_void_p)]),
    "fhpg_create_multi": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                    C.POINTER(C.c_void_p)]),
    "fhpg_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "fhpg_strips": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                              C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "fhpg_destroy": (None, [C.c_void_p]),
    "fhpg_last_error": (C.c_char_p, []),
    "fhpg_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fhpg_set_table": (C.c_int, [C.c_void_p, u8p]),
    "fhpg_set_obstacles": (C.c_int, [C.c_void_p, u8p, C.c_size_t]),
    "fhpg_upload": (C.c_int, [C.c_void_p, u8p, C.c_size_t]),
    "fhpg_download": (C.c_int, [C.c_void_p, u8p, C.c_size_t]),
    "fhpg_init": (C.c_int, [C.c_void_p, C.c_uint64, C.c_double]),
    "fhpg_advance": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, u64p]),
    "fhpg_advance_async": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64]),
    "fhpg_swaps": (C.c_int, [C.c_void_p, u64p, C.c_int]),
    "fhpg_advance_part": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int64, C.c_int]),
    "fhpg_synchronize": (C.c_int, [C.c_void_p]),
    "fhpg_bernoulli_threshold": (C.c_uint64, [C.c_double]),
    "fhpg_digest": (C.c_uint64, [C.c_void_p, C.c_size_t]),
    "fhpg_reduce_global": (C.c_int, [C.c_void_p, i64p, i64p, i64p]),
    "fhpg_reduce_cells": (C.c_int, [C.c_void_p, C.c_int, i32p, i32p, i64p, i64p]),
    "fhpg_reduce_rows": (C.c_int, [C.c_void_p, i64p, i32p]),
    "fhpg_reduce_cells_async": (C.c_int, [C.c_void_p, C.c_int]),
    "fhpg_cells_wait": (C.c_int, [C.c_void_p, i32p, i32p, i64p, i64p]),
    "fhpg_halo": (C.c_int, [C.c_void_p, vpp, vpp, vpp, vpp, C.POINTER(C.c_size_t)]),
    "fhpg_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                            C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), u64p]),
    "fhpg_force_generic": (C.c_int, [C.c_void_p, C.c_int]),
    "fhpg_select_path": (C.c_int, [C.c_void_p, C.c_int]),
    "fhpg_debug_key_span": (C.c_int, [C.c_void_p, C.c_uint32]),
    "fhpg_resident_depth": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_int)]),
    # include/fhpg_tables.h
    "fhpg_build_table": (C.c_int, [C.c_int, u8p]),
    "fhpg_validate_table": (C.c_int, [u8p, C.POINTER(C.c_int)]),
}

RULES = {"default": 0, "fhp1": 1, "fhp3": 2}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libfhpg.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run __graft_entry__.build() "
                           "(make -C paper_1208_2428_b200/csrc)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class FhpgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class FhpgInvalidArgument(FhpgError, ValueError):
    """std::invalid_argument in the reference (exit code 2)."""


def _check(rc):
    if rc != 0:
        msg = load_library().fhpg_last_error().decode()
        if rc == EINVAL:
            raise FhpgInvalidArgument(rc, msg)
        raise FhpgError(rc, msg)


def bernoulli_threshold(p: float) -> int:
    """rng.hpp:37-42 threshold (computed by the library, same double expression)."""
    return int(load_library().fhpg_bernoulli_threshold(float(p)))


def state_digest(state) -> int:
    """FNV-1a-64 of a downloaded lattice (the reference's state_digest,
    lattice.cpp:122-132), computed by the native library."""
    a = np.ascontiguousarray(state, dtype=np.uint8)
    return int(load_library().fhpg_digest(a.ctypes.data, a.nbytes))


def build_table(variant: str = "default") -> np.ndarray:
    """build_table(RuleVariant) (collision.cpp:55-72) plus FHP-I / FHP-III."""
    t = np.zeros(512, np.uint8)
    rc = load_library().fhpg_build_table(RULES.get(variant, -1), t.ctypes.data_as(u8p))
    if rc:
        raise FhpgInvalidArgument(rc, f"unknown rule variant {variant!r}")
    return t


def validate_table(table) -> int:
    """Number of validate_table issues (collision.cpp:74-101); 0 = valid."""
    t = np.ascontiguousarray(table, dtype=np.uint8)
    n = C.c_int()
    _check(load_library().fhpg_validate_table(t.ctypes.data_as(u8p), C.byref(n)))
    return n.value


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


class Engine:
    """Device-resident FHP lattice (whole lattice, or one row strip)."""

    def __init__(self, width: int, height: int, row_begin: int | None = None,
                 row_end: int | None = None, device: int | None = None,
                 strips: int | None = None, devices=None):
        """Whole lattice on the current device; a row strip [row_begin,
        row_end) on `device` (fhpg_create_strip); or, with `strips` (and
        optionally `devices`, one per strip), the whole lattice split into
        row strips over several GPUs with the halo exchange done by the
        library (fhpg_create_multi)."""
        self.lib = load_library()
        h = C.c_void_p()
        if strips is not None:
            devs = None
            if devices is not None:
                devs = (C.c_int * strips)(*[int(d) for d in devices])
                if len(devices) != strips:
                    raise ValueError("one device per strip")
            _check(self.lib.fhpg_create_multi(width, height, strips, devs, C.byref(h)))
        elif row_begin is None and row_end is None and device is None:
            _check(self.lib.fhpg_create(width, height, C.byref(h)))
        else:
            rb = 0 if row_begin is None else row_begin
            re = height if row_end is None else row_end
            dev = 0 if device is None else device
            _check(self.lib.fhpg_create_strip(width, height, rb, re, dev, C.byref(h)))
        self.h = h
        self.W, self.H = width, height
        w, hh, rb, re, fast, n = self._info()
        self.row_begin, self.row_end = rb, re
        self.nrows = re - rb

    @property
    def strips(self):
        """[(row_begin, row_end, device)] of the engine's strips."""
        n = C.c_int()
        _check(self.lib.fhpg_strips(self.h, C.byref(n), None, None, None))
        rb, re, dv = ((C.c_int * n.value)() for _ in range(3))
        _check(self.lib.fhpg_strips(self.h, C.byref(n), rb, re, dv))
        return [(rb[i], re[i], dv[i]) for i in range(n.value)]

    def _info(self):
        w, h, rb, re, fast = (C.c_int() for _ in range(5))
        n = C.c_uint64()
        _check(self.lib.fhpg_info(self.h, C.byref(w), C.byref(h), C.byref(rb), C.byref(re),
                                  C.byref(fast), C.byref(n)))
        return w.value, h.value, rb.value, re.value, fast.value, n.value

    @property
    def fast_path(self) -> bool:
        return bool(self._info()[4])

    PATHS = {0: "generic", 1: "bytes", 2: "planes"}

    @property
    def path(self) -> str:
        """Step kernel in use: "planes" (bit-plane circuit: streaming kernels,
        or for multi-step calls on small lattices the shared-memory-resident
        kernel), "bytes" (byte streaming LUT kernel) or "generic" (one thread
        per site)."""
        return self.PATHS[self._info()[4]]

    def select_path(self, path: str):
        """"auto" (default), "bytes" (no bit-plane path), "generic", or
        "streaming" (bit planes without the resident small-lattice kernel)."""
        code = {"auto": 0, "bytes": 1, "generic": 2, "streaming": 3}[path]
        _check(self.lib.fhpg_select_path(self.h, code))

    def resident_depth(self, force_p: float = 0.0) -> int:
        """Halo depth of the shared-memory-resident kernel for a multi-step
        advance at this forcing probability (0: the streaming kernels run)."""
        d = C.c_int(0)
        _check(self.lib.fhpg_resident_depth(self.h, bernoulli_threshold(force_p), C.byref(d)))
        return d.value

    @property
    def step_launches(self) -> int:
        return self._info()[5]

    def close(self):
        if getattr(self, "h", None):
            self.lib.fhpg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_stream(self, stream_ptr: int | None):
        _check(self.lib.fhpg_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def force_generic(self, on: bool = True):
        _check(self.lib.fhpg_force_generic(self.h, int(on)))

    def debug_key_span(self, rows: int = 0xFFFFFFFF):
        """Testing aid: cap the rows per column-key base of the bit-plane
        kernels (re-keying / step-key hashing past it); results unchanged."""
        _check(self.lib.fhpg_debug_key_span(self.h, rows))

    def set_table(self, table):
        t = _u8(table)
        if t.size != 512:
            raise ValueError("collision table must have 512 entries")
        _check(self.lib.fhpg_set_table(self.h, t.ctypes.data_as(u8p)))

    def set_obstacles(self, mask):
        m = _u8(mask)
        if m.shape != (self.nrows, self.W):
            raise ValueError(f"mask shape {m.shape} != {(self.nrows, self.W)}")
        _check(self.lib.fhpg_set_obstacles(self.h, m.ctypes.data_as(u8p), self.W))

    def upload(self, state):
        s = _u8(state)
        if s.shape != (self.nrows, self.W):
            raise ValueError(f"state shape {s.shape} != {(self.nrows, self.W)}")
        _check(self.lib.fhpg_upload(self.h, s.ctypes.data_as(u8p), self.W))

    def download(self, out=None):
        if out is None:
            out = np.empty((self.nrows, self.W), np.uint8)
        _check(self.lib.fhpg_download(self.h, out.ctypes.data_as(u8p), out.strides[0]))
        return out

    def init(self, seed: int, density: float):
        _check(self.lib.fhpg_init(self.h, seed, density))

    def advance(self, seed: int, force_p: float = 0.0, first_step: int = 0,
                step_count: int = 1, force_thr: int | None = None) -> int:
        thr = bernoulli_threshold(force_p) if force_thr is None else force_thr
        sw = C.c_uint64()
        _check(self.lib.fhpg_advance(self.h, seed, thr, first_step, step_count, C.byref(sw)))
        return sw.value

    def advance_async(self, seed: int, force_thr: int, first_step: int, step_count: int):
        _check(self.lib.fhpg_advance_async(self.h, seed, force_thr, first_step, step_count))

    def advance_part(self, seed: int, force_thr: int, step: int, part: int):
        """Half of one step (fhpg_advance_part): part 0 = interior rows,
        part 1 = boundary rows + buffer swap."""
        _check(self.lib.fhpg_advance_part(self.h, seed, force_thr, step, part))

    def swaps(self, reset: bool = False) -> int:
        sw = C.c_uint64()
        _check(self.lib.fhpg_swaps(self.h, C.byref(sw), int(reset)))
        return sw.value

    def synchronize(self):
        _check(self.lib.fhpg_synchronize(self.h))

    def observables(self):
        """(mass, px, py) over the engine's rows."""
        m, px, py = C.c_int64(), C.c_int64(), C.c_int64()
        _check(self.lib.fhpg_reduce_global(self.h, C.byref(m), C.byref(px), C.byref(py)))
        return m.value, px.value, py.value

    def cells(self, block: int):
        """Integer coarse-grain sums (nodes, particles, px, py), shape (cells_y, cells_x)."""
        if block < 1:
            raise FhpgInvalidArgument(EINVAL, "block size must be >= 1")
        cx, cy = (self.W + block - 1) // block, (self.H - 2 + block - 1) // block
        n = cx * cy
        nodes = np.zeros(n, np.int32)
        parts = np.zeros(n, np.int32)
        px = np.zeros(n, np.int64)
        py = np.zeros(n, np.int64)
        _check(self.lib.fhpg_reduce_cells(self.h, block, nodes.ctypes.data_as(i32p),
                                          parts.ctypes.data_as(i32p), px.ctypes.data_as(i64p),
                                          py.ctypes.data_as(i64p)))
        shp = (cy, cx)
        return nodes.reshape(shp), parts.reshape(shp), px.reshape(shp), py.reshape(shp)

    def cells_async(self, block: int):
        """Enqueue the coarse-grain sums (fhpg_reduce_cells_async); collect
        them with cells_wait(). Steps enqueued meanwhile overlap the copy."""
        _check(self.lib.fhpg_reduce_cells_async(self.h, block))
        self._cells_block = block

    def cells_wait(self):
        block = self._cells_block
        cx, cy = (self.W + block - 1) // block, (self.H - 2 + block - 1) // block
        n = cx * cy
        nodes = np.zeros(n, np.int32)
        parts = np.zeros(n, np.int32)
        px = np.zeros(n, np.int64)
        py = np.zeros(n, np.int64)
        _check(self.lib.fhpg_cells_wait(self.h, nodes.ctypes.data_as(i32p),
                                        parts.ctypes.data_as(i32p), px.ctypes.data_as(i64p),
                                        py.ctypes.data_as(i64p)))
        shp = (cy, cx)
        return nodes.reshape(shp), parts.reshape(shp), px.reshape(shp), py.reshape(shp)

    def rows(self):
        """Per interior row (index r-1): (px sum over fluid nodes, fluid count)."""
        px = np.zeros(self.H - 2, np.int64)
        fl = np.zeros(self.H - 2, np.int32)
        _check(self.lib.fhpg_reduce_rows(self.h, px.ctypes.data_as(i64p), fl.ctypes.data_as(i32p)))
        return px, fl

    def halo(self):
        """Device pointers (send_top, send_bottom, recv_top, recv_bottom), row_bytes."""
        p = [C.c_void_p() for _ in range(4)]
        n = C.c_size_t()
        _check(self.lib.fhpg_halo(self.h, *(C.byref(x) for x in p), C.byref(n)))
        return tuple(x.value for x in p), n.value
