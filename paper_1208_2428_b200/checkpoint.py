"""Checkpoint / resume of a device-resident lattice.

Same "FHPCKPT1" file as the C++ host layer (host/include/fhp_b200/checkpoint.hpp):
header (magic, width, height, next_step, seed, force_p, swaps so far, FNV-1a-64
of the state), the 512-byte table, then height x width state bytes with the
obstacle in bit 7. Exact by construction: every random draw is keyed by
(seed, purpose, step, x, y), so resuming at next_step reproduces the
uninterrupted run bit for bit.
"""
from __future__ import annotations

import dataclasses
import os
import struct

import numpy as np

MAGIC = b"FHPCKPT1"
_HEAD = struct.Struct("<8sIIqQdQQ")  # magic, W, H, next_step, seed, force_p, swaps, digest
HEADER_BYTES = _HEAD.size + 512


def _digest(state: np.ndarray) -> int:
    from .engine import state_digest
    return state_digest(state)


@dataclasses.dataclass
class Checkpoint:
    width: int
    height: int
    next_step: int
    seed: int
    force_p: float
    swaps: int
    table: np.ndarray  # 512 uint8
    state: np.ndarray  # (height, width) uint8, bit 7 = obstacle


def serialize(ck: Checkpoint, digest: int | None = None) -> bytes:
    state = np.ascontiguousarray(ck.state, dtype=np.uint8)
    if state.shape != (ck.height, ck.width):
        raise ValueError("checkpoint: state shape != (height, width)")
    table = np.ascontiguousarray(ck.table, dtype=np.uint8)
    if table.size != 512:
        raise ValueError("checkpoint: table must have 512 entries")
    if digest is None:
        digest = _digest(state)
    head = _HEAD.pack(MAGIC, ck.width, ck.height, ck.next_step, ck.seed, ck.force_p, ck.swaps,
                      digest)
    return head + table.tobytes() + state.tobytes()


def parse(data: bytes, verify: bool = True) -> Checkpoint:
    if len(data) < HEADER_BYTES or data[:8] != MAGIC:
        raise RuntimeError("checkpoint: bad magic (expected FHPCKPT1)")
    _, W, H, nxt, seed, fp, swaps, digest = _HEAD.unpack_from(data)
    if W < 1 or H < 3:
        raise RuntimeError("checkpoint: bad lattice size")
    if len(data) != HEADER_BYTES + W * H:
        raise RuntimeError("checkpoint: file size does not match width * height")
    table = np.frombuffer(data, np.uint8, 512, _HEAD.size).copy()
    state = np.frombuffer(data, np.uint8, W * H, HEADER_BYTES).reshape(H, W).copy()
    if verify and _digest(state) != digest:
        raise RuntimeError("checkpoint: state digest mismatch (corrupt file)")
    return Checkpoint(W, H, nxt, seed, fp, swaps, table, state)


def capture(engine, next_step: int, seed: int, force_p: float, swaps: int, table) -> Checkpoint:
    """Download a whole-lattice engine into a Checkpoint record (a strip
    engine holds only part of the lattice: rejected, as in checkpoint.cpp)."""
    if getattr(engine, "nrows", None) is not None and engine.nrows != engine.H:
        raise ValueError("checkpoint: engine holds a row strip, not the whole lattice")
    state = engine.download()
    H, W = state.shape
    return Checkpoint(W, H, int(next_step), int(seed), float(force_p), int(swaps),
                      np.asarray(table, np.uint8).copy(), state)


def restore(engine, ck: Checkpoint) -> None:
    """Table, obstacles (bit 7) and state back into an engine of the same size."""
    if getattr(engine, "nrows", None) is not None and (engine.nrows, engine.W) != (ck.height, ck.width):
        raise ValueError("checkpoint: engine size differs from the checkpoint's lattice")
    engine.set_table(ck.table)
    engine.set_obstacles((ck.state >> 7).astype(np.uint8))
    engine.upload(ck.state)


def save(path: str, ck: Checkpoint, digest: int | None = None) -> None:
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(serialize(ck, digest))
    os.replace(tmp, path)


def load(path: str, verify: bool = True) -> Checkpoint:
    with open(path, "rb") as f:
        return parse(f.read(), verify)
