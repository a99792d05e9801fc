"""Python mirror of the reference pentadiagonal API (stengrid/penta.hpp:12-123).

``PentaBatch`` / ``RhsBatch`` keep the reference's interleaved layout
(entry (system b, row r) at ``r*batchCount + b``, penta.hpp:12-32), exposed as
numpy arrays of shape (n, batchCount). ``PentaFactor`` / ``PeriodicPentaFactor``
factor ON THE DEVICE (one system per thread, sm_100a) and solve in place;
zero pivots raise ``PentaSolveError`` with the reference's system index.
``interleave`` / ``deinterleave`` are pure layout moves (penta.cpp:337-384).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import InvalidArgument, check


def _check_shapes(batch_count, n):  # penta.cpp:10-13
    if batch_count < 1:
        raise InvalidArgument("penta: batchCount must be >= 1")
    if n < 5:
        raise InvalidArgument("penta: systems need n >= 5")


class PentaBatch:
    """penta.hpp:21-33 — five bands, interleaved, shape (n, batchCount)."""

    def __init__(self, batch_count: int, n: int, periodic: bool):
        _check_shapes(batch_count, n)
        self.batchCount, self.n, self.periodic = batch_count, n, bool(periodic)
        z = lambda: np.zeros((n, batch_count))
        self.secondSub, self.sub, self.diag, self.super, self.secondSuper = z(), z(), z(), z(), z()

    def idx(self, b, r):
        return r * self.batchCount + b

    def bands(self):
        return (self.secondSub, self.sub, self.diag, self.super, self.secondSuper)


class RhsBatch:
    """penta.hpp:36-49."""

    def __init__(self, batch_count: int, n: int, values=None):
        if batch_count < 1 or n < 1:
            raise InvalidArgument("RhsBatch: batchCount and n must be >= 1")
        self.batchCount, self.n = batch_count, n
        self.values = np.zeros((n, batch_count)) if values is None else np.ascontiguousarray(values, dtype=np.float64)

    def at(self, b, r):
        return self.values[r, b]


class _DeviceFactor:
    periodic = False

    def __init__(self, m: PentaBatch):
        _check_shapes(m.batchCount, m.n)
        self._h = C.c_void_p()
        self.B, self.n_ = m.batchCount, m.n
        bands = [np.ascontiguousarray(x, dtype=np.float64) for x in m.bands()]
        check(_lib.lib().sg_penta_create(m.batchCount, m.n, int(self.periodic),
                                         *(C.c_void_p(x.ctypes.data) for x in bands), 0, C.byref(self._h)))

    def batch_count(self):
        return self.B

    def size(self):
        return self.n_

    def solve_in_place(self, rhs, pool=None):
        """penta.cpp:199-202 / 289-295. ``rhs`` is a RhsBatch (host) or a
        CUDA tensor of shape (n, B) (device, zero-copy)."""
        if isinstance(rhs, RhsBatch):
            if rhs.batchCount != self.B or rhs.n != self.n_:
                who = "PeriodicPentaFactor" if self.periodic else "PentaFactor"
                raise InvalidArgument(f"{who}::solve_in_place: rhs shape does not match the operator")
            check(_lib.lib().sg_penta_solve(self._h, C.c_void_p(rhs.values.ctypes.data), 0, None, 1))
        else:
            if tuple(rhs.shape) != (self.n_, self.B) or not rhs.is_contiguous():
                raise InvalidArgument("solve_in_place: rhs shape does not match the operator")
            # in order with the caller's torch stream
            import torch
            stream = torch.cuda.current_stream(rhs.device).cuda_stream
            check(_lib.lib().sg_penta_solve(self._h, C.c_void_p(rhs.data_ptr()), 1, C.c_void_p(stream or 0), 1))

    def __del__(self):
        try:
            if self._h.value:
                _lib.lib().sg_penta_destroy(C.byref(self._h))
        except Exception:
            pass


class PentaFactor(_DeviceFactor):
    """penta.hpp:57-77 (non-periodic bands; wrap slots ignored)."""
    periodic = False


class PeriodicPentaFactor(_DeviceFactor):
    """penta.hpp:79-100 (Woodbury corner correction)."""
    periodic = True


def solve_batch(m: PentaBatch, rhs: RhsBatch, pool=None) -> RhsBatch:
    """penta.cpp:297-303."""
    if m.periodic:
        raise InvalidArgument("solve_batch: operator is periodic")
    if rhs.batchCount != m.batchCount or rhs.n != m.n:
        raise InvalidArgument("solve_batch: rhs shape does not match the operator")
    out = RhsBatch(rhs.batchCount, rhs.n, rhs.values.copy())
    PentaFactor(m).solve_in_place(out, pool)
    return out


def solve_periodic_batch(m: PentaBatch, rhs: RhsBatch, pool=None) -> RhsBatch:
    """penta.cpp:305-311."""
    if not m.periodic:
        raise InvalidArgument("solve_periodic_batch: operator is not periodic")
    if rhs.batchCount != m.batchCount or rhs.n != m.n:
        raise InvalidArgument("solve_periodic_batch: rhs shape does not match the operator")
    out = RhsBatch(rhs.batchCount, rhs.n, rhs.values.copy())
    PeriodicPentaFactor(m).solve_in_place(out, pool)
    return out


def build_hyperdiffusion_operator(sigma: float, n: int, batch_count: int, periodic: bool) -> PentaBatch:
    """penta.cpp:313-335 — rows {s, -4s, 1+6s, -4s, s}."""
    if not (sigma >= 0.0):
        raise InvalidArgument("build_hyperdiffusion_operator: sigma must be >= 0")
    m = PentaBatch(batch_count, n, periodic)
    first = -4.0 * sigma
    center = 1.0 + 6.0 * sigma
    m.secondSub[:] = sigma
    m.sub[:] = first
    m.diag[:] = center
    m.super[:] = first
    m.secondSuper[:] = sigma
    if not periodic:
        m.secondSub[0, :] = 0.0
        m.secondSub[1, :] = 0.0
        m.sub[0, :] = 0.0
        m.super[n - 1, :] = 0.0
        m.secondSuper[n - 2, :] = 0.0
        m.secondSuper[n - 1, :] = 0.0
    return m


class Axis:
    X = 0
    Y = 1


def interleave(g, axis) -> RhsBatch:
    """penta.cpp:337-360 — Axis.X: one system per row (transposed copy)."""
    v = g.values
    if axis == Axis.X:
        return RhsBatch(g.ny, g.nx, np.ascontiguousarray(v.T))
    return RhsBatch(g.nx, g.ny, v.copy())


def deinterleave(rhs: RhsBatch, axis, dx, dy):
    """penta.cpp:362-384."""
    from .stencil import Grid2D
    if axis == Axis.X:
        g = Grid2D(rhs.n, rhs.batchCount, dx, dy)
        g.values = np.ascontiguousarray(rhs.values.T)
    else:
        g = Grid2D(rhs.batchCount, rhs.n, dx, dy)
        g.values = rhs.values.copy()
    return g
