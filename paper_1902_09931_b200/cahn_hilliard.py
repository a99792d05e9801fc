"""Python mirror of the reference Cahn-Hilliard API (stengrid/cahn_hilliard.hpp).

``CHStepper`` runs the BDF2-ADI step entirely on the GPU (csrc/ch.cu: fused
RHS kernel, two batched cyclic pentadiagonal sweeps with fused Woodbury
corrections, CUDA-graph replay); host fields are only touched by
``set_state`` / ``field()``. Fields are bitwise identical to the reference
``CHStepper`` on the same parameters.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import InvalidArgument, SgChParams, check
from .stencil import Grid2D

TWO_PI = 2.0 * math.pi


@dataclass
class CHParams:
    """cahn_hilliard.hpp:23-39 (defaults identical)."""
    D: float = 1.0
    gamma: float = 0.01
    nx: int = 512
    ny: int = 512
    lx: float = TWO_PI
    ly: float = TWO_PI
    dt: float = 0.0
    T: float = 0.0
    seed: int = 1
    icAmplitude: float = 0.1
    nonlinearEnabled: bool = True

    def dx(self) -> float:
        return self.lx / self.nx

    def dy(self) -> float:
        return self.ly / self.ny

    def _c(self) -> SgChParams:
        return SgChParams(self.D, self.gamma, self.lx, self.ly, self.dt, self.T, self.icAmplitude,
                          self.nx, self.ny, self.seed, int(self.nonlinearEnabled))

    def validate(self) -> None:
        """cahn_hilliard.cpp:56-66."""
        p = self._c()
        check(_lib.lib().sg_ch_validate(C.byref(p)))


@dataclass
class Diagnostics:
    t: float = 0.0
    s: float = 0.0
    k1Inv: float = 0.0


def nonlinear_laplacian_coefficients(dx: float, dy: float):
    """cahn_hilliard.cpp:78-83."""
    cx = 1.0 / (dx * dx)
    cy = 1.0 / (dy * dy)
    cc = -2.0 * cx - 2.0 * cy
    return [0.0, cy, 0.0, cx, cc, cx, 0.0, cy, 0.0]


def biharmonic_weights(dx: float, dy: float):
    """cahn_hilliard.cpp:85-114 (same accumulation order; the last non-zero
    entry absorbs the row-major prefix residual so the sum is exactly 0)."""
    def pow4(h):
        h2 = h * h
        return h2 * h2
    ax = 1.0 / pow4(dx)
    ay = 1.0 / pow4(dy)
    cr = 2.0 / ((dx * dx) * (dy * dy))
    w = [0.0] * 25

    def add(p, q, v):
        w[q * 5 + p] = w[q * 5 + p] + v
    add(0, 2, ax); add(1, 2, -4.0 * ax); add(2, 2, 6.0 * ax); add(3, 2, -4.0 * ax); add(4, 2, ax)
    add(2, 0, ay); add(2, 1, -4.0 * ay); add(2, 2, 6.0 * ay); add(2, 3, -4.0 * ay); add(2, 4, ay)
    cross = [1.0, -2.0, 1.0, -2.0, 4.0, -2.0, 1.0, -2.0, 1.0]
    for q in range(3):
        for p in range(3):
            add(p + 1, q + 1, cross[q * 3 + p] * cr)
    prefix = 0.0
    for k in range(22):
        prefix = prefix + w[k]
    w[4 * 5 + 2] = -prefix
    return w


def _field_ptr(g):
    """(pointer, memory kind, nx, ny, dx, dy) of a Grid2D or 2D CUDA tensor."""
    if isinstance(g, Grid2D):
        v = np.ascontiguousarray(g.values, dtype=np.float64)
        return v, C.c_void_p(v.ctypes.data), 0, g.nx, g.ny, g.dx, g.dy
    # a CUDA tensor: its producer may still run on the caller's torch stream
    import torch
    torch.cuda.current_stream(g.device).synchronize()
    return g, C.c_void_p(g.data_ptr()), 1, int(g.shape[1]), int(g.shape[0]), 1.0, 1.0


def simpson_mean(g) -> float:
    """cahn_hilliard.cpp:161-177 on the device (bitwise identical)."""
    keep, ptr, mem, nx, ny, _, _ = _field_ptr(g)
    out = C.c_double()
    check(_lib.lib().sg_simpson_mean(ptr, nx, ny, 0, mem, C.byref(out)))
    return out.value


def s_metric(g) -> float:
    """cahn_hilliard.cpp:179-188 on the device; DomainError when saturated."""
    keep, ptr, mem, nx, ny, _, _ = _field_ptr(g)
    out = C.c_double()
    check(_lib.lib().sg_s_metric(ptr, nx, ny, mem, C.byref(out)))
    return out.value


def k1_metric(g, dx=None, dy=None) -> float:
    """cahn_hilliard.cpp:190-211 on the device (cuFFT); DomainError on zero."""
    keep, ptr, mem, nx, ny, gdx, gdy = _field_ptr(g)
    out = C.c_double()
    check(_lib.lib().sg_k1_metric(ptr, nx, ny, dx or gdx, dy or gdy, mem, C.byref(out)))
    return out.value


class CHStepper:
    """cahn_hilliard.hpp:104-137 — state lives in HBM."""

    def __init__(self, params: CHParams, num_tiles: int = 1, num_workers: int = 1):
        self._h = C.c_void_p()
        self._p = params
        cp = params._c()
        check(_lib.lib().sg_ch_create(C.byref(cp), num_tiles, num_workers, C.byref(self._h)))

    def params(self) -> CHParams:
        return self._p

    def step(self) -> None:
        check(_lib.lib().sg_ch_step(self._h, 1))

    def step_many(self, steps: int) -> None:
        """`steps` consecutive step() calls, enqueued without host syncs."""
        check(_lib.lib().sg_ch_step(self._h, int(steps)))

    def synchronize(self) -> None:
        check(_lib.lib().sg_ch_synchronize(self._h))

    def set_partition(self, segments: int) -> None:
        """Extension (sg_ch_set_partition): partitioned x/y sweeps with
        ``segments`` segments per system (>= 2; 0/1 = the bitwise default).
        Not bitwise equal to the reference; see DESIGN.md for the measured
        deviation."""
        check(_lib.lib().sg_ch_set_partition(self._h, int(segments)))

    def workers(self):
        """(GPU count, P2P form?) — numWorkers -> GPUs (sg_ch_workers)."""
        n, p2p = C.c_int(), C.c_int()
        check(_lib.lib().sg_ch_workers(self._h, C.byref(n), C.byref(p2p)))
        return n.value, bool(p2p.value)

    def set_state(self, curr: Grid2D, prev: Grid2D) -> None:
        """cahn_hilliard.cpp:251-258."""
        p = self._p
        if curr.nx != p.nx or curr.ny != p.ny or not curr.same_shape(prev):
            raise InvalidArgument("CHStepper::set_state: shape mismatch")
        c = np.ascontiguousarray(curr.values, dtype=np.float64)
        q = np.ascontiguousarray(prev.values, dtype=np.float64)
        check(_lib.lib().sg_ch_set_state(self._h, C.c_void_p(c.ctypes.data), C.c_void_p(q.ctypes.data), 0))

    def _get(self, which) -> Grid2D:
        p = self._p
        g = Grid2D(p.nx, p.ny, p.dx(), p.dy())
        check(_lib.lib().sg_ch_get_field(self._h, which, C.c_void_p(g.values.ctypes.data), 0))
        return g

    def field(self) -> Grid2D:
        return self._get(0)

    def previous_field(self) -> Grid2D:
        return self._get(1)

    def device_field_ptr(self, which: int = 0) -> int:
        ptr = C.c_void_p()
        check(_lib.lib().sg_ch_device_field(self._h, which, C.byref(ptr)))
        return ptr.value

    def diagnostics(self) -> Diagnostics:
        """cahn_hilliard.cpp:330-340, computed on the device-resident C^n."""
        t, s_, k = C.c_double(), C.c_double(), C.c_double()
        check(_lib.lib().sg_ch_diagnostics(self._h, C.byref(t), C.byref(s_), C.byref(k)))
        return Diagnostics(t.value, s_.value, k.value)

    def step_index(self) -> int:
        s = C.c_int()
        check(_lib.lib().sg_ch_status(self._h, C.byref(s), None))
        return s.value

    def time(self) -> float:
        t = C.c_double()
        check(_lib.lib().sg_ch_status(self._h, None, C.byref(t)))
        return t.value

    def __del__(self):
        try:
            if self._h.value:
                _lib.lib().sg_ch_destroy(C.byref(self._h))
        except Exception:
            pass


@dataclass
class RunSink:
    """cahn_hilliard.hpp:141-146."""
    diagEvery: int = 1
    snapEvery: int = 0
    onDiagnostics: object = None
    onSnapshot: object = None


def run(params: CHParams, num_tiles: int, num_workers: int, sink: RunSink) -> None:
    """cahn_hilliard.cpp:342-356: step to T (ceil(T/dt - 1e-9) steps),
    emitting diagnostics / snapshots at the sink cadences; steps between
    emissions are enqueued back to back on the device."""
    import math as _m
    st = CHStepper(params, num_tiles, num_workers)

    def emit(step):
        if sink.diagEvery > 0 and sink.onDiagnostics and step % sink.diagEvery == 0:
            sink.onDiagnostics(st.diagnostics())
        if sink.snapEvery > 0 and sink.onSnapshot and step % sink.snapEvery == 0:
            sink.onSnapshot(st.field(), step, st.time())

    emit(0)
    steps = int(_m.ceil(params.T / params.dt - 1e-9))
    cadences = [c for c, f in ((sink.diagEvery, sink.onDiagnostics), (sink.snapEvery, sink.onSnapshot))
                if c > 0 and f]
    s = 0
    while s < steps:
        nxt = steps
        for c in cadences:
            nxt = min(nxt, (s // c + 1) * c)
        st.step_many(nxt - s)
        s = nxt
        emit(s)
