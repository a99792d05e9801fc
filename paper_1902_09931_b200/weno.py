"""Python mirror of the reference WENO5 advection API (stengrid/weno.hpp).

``weno_advect`` runs on the device (csrc/weno.cu), bitwise identical to the
reference; ``weno_derivative_7`` / ``upwind_side`` are the reference's scalar
helpers (weno.cpp:13-48), kept for API completeness.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import InvalidArgument, check
from .stencil import Grid2D

WENO_EPS = 1e-6


@dataclass
class VelocityField:
    u: Grid2D
    v: Grid2D


class UpwindSide:
    Left = 0
    Right = 1


def upwind_side(velocity: float) -> int:
    """weno.hpp:15-17."""
    return UpwindSide.Right if velocity < 0.0 else UpwindSide.Left


def _combine(v1, v2, v3, v4, v5):  # weno.cpp:13-29
    c1 = v1 * (1.0 / 3.0) - v2 * (7.0 / 6.0) + v3 * (11.0 / 6.0)
    c2 = -v2 * (1.0 / 6.0) + v3 * (5.0 / 6.0) + v4 * (1.0 / 3.0)
    c3 = v3 * (1.0 / 3.0) + v4 * (5.0 / 6.0) - v5 * (1.0 / 6.0)
    d1 = v1 - 2.0 * v2 + v3
    d2 = v2 - 2.0 * v3 + v4
    d3 = v3 - 2.0 * v4 + v5
    s1 = (13.0 / 12.0) * d1 * d1 + 0.25 * (v1 - 4.0 * v2 + 3.0 * v3) * (v1 - 4.0 * v2 + 3.0 * v3)
    s2 = (13.0 / 12.0) * d2 * d2 + 0.25 * (v2 - v4) * (v2 - v4)
    s3 = (13.0 / 12.0) * d3 * d3 + 0.25 * (3.0 * v3 - 4.0 * v4 + v5) * (3.0 * v3 - 4.0 * v4 + v5)
    a1 = 0.1 / ((WENO_EPS + s1) * (WENO_EPS + s1))
    a2 = 0.6 / ((WENO_EPS + s2) * (WENO_EPS + s2))
    a3 = 0.3 / ((WENO_EPS + s3) * (WENO_EPS + s3))
    return (a1 * c1 + a2 * c2 + a3 * c3) / (a1 + a2 + a3)


def weno_derivative_7(w7, inv_h: float, side: int) -> float:
    """weno.cpp:33-48 (scalar helper)."""
    w = [float(x) for x in w7]
    if side == UpwindSide.Left:
        return _combine(*[(w[k + 1] - w[k]) * inv_h for k in range(5)])
    return _combine(*[(w[6 - k] - w[5 - k]) * inv_h for k in range(5)])


def weno_advect(phi: Grid2D, vel: VelocityField, num_tiles: int = 1, num_workers: int = 1) -> Grid2D:
    """weno.cpp:50-94 on the GPU."""
    if not phi.same_shape(vel.u) or not phi.same_shape(vel.v):
        raise InvalidArgument("weno_advect: velocity shape does not match the field")
    if num_tiles < 1 or num_tiles > phi.ny:
        raise InvalidArgument("make_tiles: numTiles must satisfy 1 <= numTiles <= ny")
    if num_workers < 1:
        raise InvalidArgument("WorkerPool: workers must be >= 1")
    f = np.ascontiguousarray(phi.values, dtype=np.float64)
    u = np.ascontiguousarray(vel.u.values, dtype=np.float64)
    v = np.ascontiguousarray(vel.v.values, dtype=np.float64)
    out = Grid2D(phi.nx, phi.ny, phi.dx, phi.dy) if phi.nx >= 1 else None
    p = lambda a: C.c_void_p(a.ctypes.data)
    check(_lib.lib().sg_weno_advect(p(f), p(u), p(v), phi.nx, phi.ny, phi.dx, phi.dy, p(out.values), 0, None))
    return out
