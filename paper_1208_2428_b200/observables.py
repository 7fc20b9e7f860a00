"""Observable finalisation on the host (integer sums come from the device).

The device reductions (fhpg_reduce_cells / fhpg_reduce_rows) return exact
integer sums; the floating-point finalisation below uses the reference's
expressions operation for operation so the doubles are bit-identical:

* coarse_grain   observables.cpp:49-82 (rho = particles/nodes,
                 ux = px*0.5/max(particles,1), uy = py*0.8660254037844386/max(...))
* velocity_profile observables.cpp:84-102 (mean_ux = px/2.0/count)
* writers        observables.cpp:104-149 (CSV, PGM)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

K_SQRT3_HALF = 0.8660254037844386  # observables.cpp:10


@dataclass
class FlowField:
    """observables.hpp:21-37; arrays of shape (cells_y, cells_x)."""
    block: int
    nodes: np.ndarray
    particles: np.ndarray
    rho: np.ndarray
    ux: np.ndarray
    uy: np.ndarray

    @property
    def cells_x(self):
        return self.nodes.shape[1]

    @property
    def cells_y(self):
        return self.nodes.shape[0]


def finalize_cells(block, nodes, particles, px, py) -> FlowField:
    nodes = np.asarray(nodes, np.int32)
    particles = np.asarray(particles, np.int32)
    px = np.asarray(px, np.int64)
    py = np.asarray(py, np.int64)
    with np.errstate(invalid="ignore", divide="ignore"):
        rho = np.where(nodes > 0, particles.astype(np.float64) / np.maximum(nodes, 1), 0.0)
    denom = np.maximum(particles, 1).astype(np.float64)
    # ux_of(p) = p.px * 0.5 (int -> double, then multiply), then / denom.
    ux = (px.astype(np.float64) * 0.5) / denom
    uy = (py.astype(np.float64) * K_SQRT3_HALF) / denom
    return FlowField(block, nodes, particles, rho, ux, uy)


def finalize_profile(px_rows, fluid_rows):
    """(rows, mean_ux, sample_count) for interior rows 1..H-2."""
    px = np.asarray(px_rows, np.int64)
    n = np.asarray(fluid_rows, np.int32)
    with np.errstate(invalid="ignore", divide="ignore"):
        mean = np.where(n > 0, px.astype(np.float64) / 2.0 / np.maximum(n, 1), 0.0)
    rows = np.arange(1, px.size + 1)
    return rows, mean, n


def coarse_grain(engine, block: int) -> FlowField:
    """coarse_grain(lat, block) on a device-resident lattice."""
    return finalize_cells(block, *engine.cells(block))


def velocity_profile(engine):
    return finalize_profile(*engine.rows())


def _fmt(v: float) -> str:
    # std::ostream default formatting (%g with 6 significant digits).
    return "%g" % v


def write_flow_csv(path, field: FlowField):
    """observables.cpp:104-114."""
    with open(path, "w") as f:
        f.write("cell_x,cell_y,rho,ux,uy\n")
        for cy in range(field.cells_y):
            for cx in range(field.cells_x):
                f.write(f"{cx},{cy},{_fmt(field.rho[cy, cx])},{_fmt(field.ux[cy, cx])},"
                        f"{_fmt(field.uy[cy, cx])}\n")


def write_profile_csv(path, rows, mean_ux, count):
    """observables.cpp:116-122."""
    with open(path, "w") as f:
        f.write("row,mean_ux,sample_count\n")
        for r, m, n in zip(rows, mean_ux, count):
            f.write(f"{r},{_fmt(m)},{n}\n")


def write_density_pgm(path, field: FlowField):
    """observables.cpp:124-133: P5, pixel = lround(255*rho/7) clamped."""
    v = np.clip(np.floor(255.0 * field.rho / 7.0 + 0.5), 0, 255).astype(np.uint8)
    with open(path, "wb") as f:
        f.write(f"P5\n{field.cells_x} {field.cells_y}\n255\n".encode())
        f.write(v.tobytes())
