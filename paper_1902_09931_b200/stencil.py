"""Python mirror of the reference stencil API (stengrid/stencil.hpp:12-114).

Same names, argument meaning and error behaviour as the reference C++ API:
``create_plan`` / ``compute`` / ``swap_plan`` / ``destroy_plan`` over
``Grid2D`` fields, ``WeightStencil`` / ``FunctionStencil`` kinds, the
``Direction`` / ``BoundaryMode`` / ``Residency`` enums. Exceptions are the
Python twins of the reference's: ``InvalidArgument`` (std::invalid_argument)
and ``LogicError`` (std::logic_error).

All arithmetic runs in the sm_100a kernels of libstengrid_b200.so through the
C ABI (include/stengrid/sg.h). Grids are either host ``Grid2D`` objects
(numpy storage; the plan mirrors them on the device and moves data according
to ``Residency``) or CUDA ``torch.Tensor``s (zero-copy, device-resident).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Sequence, Union

import numpy as np

from . import _lib
from ._lib import FUNCTIONS, InvalidArgument, LogicError, SgExtents, SgSlabDesc, check


class Direction(IntEnum):
    X = 0
    Y = 1
    XY = 2


class BoundaryMode(IntEnum):
    Periodic = 0
    NonPeriodic = 1


class Residency(IntEnum):
    Host = 0
    Device = 1


@dataclass
class Extents:
    """grid.hpp:53-62 — how far the window reaches from its point."""
    left: int = 0
    right: int = 0
    top: int = 0
    bottom: int = 0

    def width(self) -> int:
        return self.left + self.right + 1

    def height(self) -> int:
        return self.top + self.bottom + 1

    def valid(self) -> bool:
        return min(self.left, self.right, self.top, self.bottom) >= 0

    def _c(self) -> SgExtents:
        return SgExtents(self.left, self.right, self.top, self.bottom)


@dataclass
class WeightStencil:
    """stencil.hpp:12-18 — row-major W*H weights, origin top-left."""
    ext: Extents
    weights: Sequence[float]


@dataclass
class FunctionStencil:
    """stencil.hpp:29-33 — a window function plus coefficients. ``fn`` names
    one of the device window functions (``FUNCTIONS``) — the device twin of
    the reference's host function pointer — or a function registered from
    source (``register_function_source``). ``None`` is the null pointer."""
    ext: Extents
    fn: Union[str, int, None]
    coe: Sequence[float] = field(default_factory=list)


class Grid2D:
    """grid.hpp:25-49 — a uniform 2D field; ``values[j, i]`` is sample (i, j)."""

    def __init__(self, nx: int, ny: int, dx: float = 1.0, dy: float = 1.0, dtype=np.float64):
        if nx < 1 or ny < 1:
            raise InvalidArgument("Grid2D: nx and ny must be >= 1")
        if not (dx > 0.0) or not (dy > 0.0):
            raise InvalidArgument("Grid2D: dx and dy must be > 0")
        self.nx, self.ny, self.dx, self.dy = nx, ny, dx, dy
        self.values = np.zeros((ny, nx), dtype=dtype)

    @classmethod
    def from_array(cls, arr, dx=1.0, dy=1.0):
        a = np.ascontiguousarray(arr)
        g = cls(a.shape[1], a.shape[0], dx, dy, dtype=a.dtype)
        g.values = a
        return g

    def __call__(self, i, j):
        return self.values[j, i]

    def same_shape(self, other) -> bool:
        return self.nx == other.nx and self.ny == other.ny

    def copy(self):
        g = Grid2D(self.nx, self.ny, self.dx, self.dy, dtype=self.values.dtype)
        g.values = self.values.copy()
        return g


def _current_stream():
    import torch
    return torch.cuda.current_stream().cuda_stream


def _dtype_code(dt) -> int:
    s = str(dt)
    if s.endswith("float64"):
        return 0
    if s.endswith("float32"):
        return 1
    raise InvalidArgument(f"stengrid: unsupported dtype {dt} (float64 or float32)")


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _shape(x):
    if isinstance(x, Grid2D):
        return x.nx, x.ny
    if _is_torch_cuda(x) and x.dim() == 2:
        return int(x.shape[1]), int(x.shape[0])
    raise InvalidArgument("stengrid: grids are Grid2D (host) or 2D CUDA tensors (device)")


# name -> id of the functions registered from source (register_function_source)
SOURCE_FUNCTIONS: dict = {}


def register_function_source(name: str, body: str) -> int:
    """Register a window function from CUDA C++ source (sg.h:
    sg_register_function_source). ``body`` is the body of
    ``T fn(const T* window, const T* coe, int rowStride)`` — the reference's
    StencilFunction contract (stencil.hpp:20-25), entry (p, q) at
    ``window[q*rowStride + p]``. Compiled by NVRTC (sm_100a, no FMA
    contraction) into the library's stencil kernels on first use. Returns the
    function id; ``FunctionStencil(ext, name, coe)`` then selects it.
    Raises InvalidArgument (with the compiler log) if the body does not
    compile."""
    fid = C.c_int(-1)
    check(_lib.lib().sg_register_function_source(name.encode(), body.encode(), C.byref(fid)))
    SOURCE_FUNCTIONS[name] = fid.value
    return fid.value


def _kind_values(kind):
    if isinstance(kind, WeightStencil):
        return 0, np.ascontiguousarray(np.asarray(kind.weights, dtype=np.float64))
    if isinstance(kind, FunctionStencil):
        fn = kind.fn
        if fn is None:
            fid = -1
        elif isinstance(fn, str):
            if fn in SOURCE_FUNCTIONS:
                fid = SOURCE_FUNCTIONS[fn]
            elif fn in FUNCTIONS:
                fid = FUNCTIONS[fn]
            else:
                raise InvalidArgument(f"create_plan: no device twin registered for function {fn!r}")
        else:
            fid = int(fn)
        return fid, np.ascontiguousarray(np.asarray(kind.coe, dtype=np.float64))
    raise InvalidArgument("create_plan: kind must be WeightStencil or FunctionStencil")


class StencilPlan:
    """stencil.hpp:42-85 — movable, never owns the fields."""

    def __init__(self):
        self._h = C.c_void_p()
        self._grids = [None, None]
        self._in = 0
        self.direction = Direction.X
        self.mode = BoundaryMode.Periodic
        self.ext = Extents()
        self._tiles = []
        self.num_workers = 1
        self._device = False

    def valid(self) -> bool:
        return bool(self._h.value) and _lib.lib().sg_plan_valid(self._h) == 1

    def extents(self):
        return self.ext

    def tiles(self):
        return list(self._tiles)

    def input(self):
        return self._grids[self._in] if self.valid() else None

    def output(self):
        return self._grids[1 - self._in] if self.valid() else None

    def kernel_kind(self) -> int:
        return _lib.lib().sg_plan_kernel_kind(self._h)

    def workers(self):
        """[(device, row_begin, row_end)] of the plan's workers (numWorkers
        -> GPUs for host grids; one entry for a one-GPU plan)."""
        n = C.c_int()
        check(_lib.lib().sg_plan_workers(self._h, C.byref(n), None, None, None, 0))
        dev, b, e = ((C.c_int * n.value)() for _ in range(3))
        check(_lib.lib().sg_plan_workers(self._h, C.byref(n), dev, b, e, n.value))
        return [(dev[k], b[k], e[k]) for k in range(n.value)]

    def destroy(self):
        if self._h.value:
            check(_lib.lib().sg_plan_destroy(C.byref(self._h)))
        self._grids = [None, None]
        self._tiles = []

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def set_device_map(mode: str) -> None:
    """How numWorkers maps to GPUs (sg_set_device_map): "clip" (default) —
    min(numWorkers, visible GPUs) workers; "modulo" — numWorkers workers,
    worker w on GPU w % visible GPUs (tests on a one-GPU box)."""
    modes = {"clip": 0, "modulo": 1}
    if mode not in modes:
        raise InvalidArgument("set_device_map: mode must be 'clip' or 'modulo'")
    check(_lib.lib().sg_set_device_map(modes[mode]))


def get_device_map() -> str:
    return ("clip", "modulo")[_lib.lib().sg_get_device_map()]


def make_tiles(ny: int, num_tiles: int):
    """grid.cpp:62-82 — contiguous row ranges, larger tiles first."""
    b = (C.c_int * max(num_tiles, 1))()
    e = (C.c_int * max(num_tiles, 1))()
    check(_lib.lib().sg_make_tiles(ny, num_tiles, b, e))
    return [(b[k], e[k]) for k in range(num_tiles)]


def wrap(i: int, n: int) -> int:
    """grid.cpp:42-47."""
    out = C.c_int()
    check(_lib.lib().sg_wrap(i, n, C.byref(out)))
    return out.value


def create_plan(direction, mode, kind, input, output, num_tiles: int = 1, num_workers: int = 1,
                shared_pool=None) -> StencilPlan:
    """stencil.hpp:90-92 / stencil.cpp:152-184."""
    nxi, nyi = _shape(input)
    nxo, nyo = _shape(output)
    if (nxi, nyi) != (nxo, nyo):
        raise InvalidArgument("create_plan: input and output shapes differ")
    if shared_pool is not None and getattr(shared_pool, "workers", lambda: num_workers)() != num_workers:
        raise InvalidArgument("create_plan: shared pool size does not match numWorkers")
    host = isinstance(input, Grid2D)
    if host != isinstance(output, Grid2D):
        raise InvalidArgument("create_plan: input and output must both be host or both device grids")
    if host:
        if input is output or input.values.ctypes.data == output.values.ctypes.data:
            raise InvalidArgument("create_plan: input and output must be distinct buffers")
        if input.values.dtype != output.values.dtype:
            raise InvalidArgument("create_plan: input and output dtypes differ")
        for g in (input, output):
            if not g.values.flags.c_contiguous:
                g.values = np.ascontiguousarray(g.values)
        pin, pout = input.values.ctypes.data, output.values.ctypes.data
        dtype = _dtype_code(input.values.dtype)
        memory = 0
    else:
        if input.data_ptr() == output.data_ptr():
            raise InvalidArgument("create_plan: input and output must be distinct buffers")
        if not (input.is_contiguous() and output.is_contiguous()) or input.dtype != output.dtype:
            raise InvalidArgument("create_plan: device grids must be contiguous and share a dtype")
        pin, pout = input.data_ptr(), output.data_ptr()
        dtype = _dtype_code(input.dtype)
        memory = 1
    fid, vals = _kind_values(kind)
    ext = kind.ext
    plan = StencilPlan()
    vptr = vals.ctypes.data_as(C.POINTER(C.c_double)) if vals.size else None
    check(_lib.lib().sg_plan_create(int(direction), int(mode), ext._c(), fid, vptr, vals.size, dtype,
                                    C.c_void_p(pin), C.c_void_p(pout), nxi, nyi, memory, num_tiles,
                                    num_workers, C.byref(plan._h)))
    plan._grids = [input, output]
    plan._device = not host
    plan.direction, plan.mode, plan.ext = Direction(direction), BoundaryMode(mode), ext
    plan._tiles = make_tiles(nyi, num_tiles)
    plan.num_workers = num_workers
    return plan


def destroy_plan(plan: StencilPlan) -> None:
    """stencil.cpp:186-195 — idempotent; never touches the grids."""
    plan.destroy()


def swap_plan(plan: StencilPlan) -> None:
    """stencil.cpp:197-200."""
    if not plan.valid():
        raise LogicError("swap_plan: plan was destroyed")
    check(_lib.lib().sg_plan_swap(plan._h))
    plan._in = 1 - plan._in


def compute(plan: StencilPlan, hint: Residency = Residency.Host, stream=None,
            synchronize=None) -> None:
    """stencil.cpp:202-235 — apply the stencil on the GPU.

    Host-bound plans: ``Residency.Host`` leaves the host output valid on
    return; ``Residency.Device`` keeps it on the device until
    :func:`sync_to_host`. ``stream`` is a ``torch.cuda.Stream`` / raw
    cudaStream_t or None (the plan's own stream). ``synchronize`` defaults to
    ``hint == Residency.Host``: Device-residency applications return once
    queued."""
    if synchronize is None:
        synchronize = hint == Residency.Host
    if not plan.valid():
        raise LogicError("compute: plan was destroyed")
    s = getattr(stream, "cuda_stream", stream)
    if s is None and plan._device:
        # device grids (torch tensors): run in order with the caller's work
        s = _current_stream()
    check(_lib.lib().sg_plan_compute(plan._h, int(hint), C.c_void_p(s or 0), int(bool(synchronize))))


def sync_to_host(plan: StencilPlan) -> None:
    check(_lib.lib().sg_plan_sync_to_host(plan._h))


def mark_host_dirty(plan: StencilPlan, which: int) -> None:
    check(_lib.lib().sg_plan_mark_host_dirty(plan._h, which))


def launch_slab(desc: dict, ext: Extents, kind, inp, out, stream=None, peers=None) -> None:
    """Stateless device launch over a y-slab (sg_stencil_launch): computes
    output rows [row0,row1) × cols [col0,col1); input row for output row j,
    tap q is j + inShift - top + q (wrapped modulo inRows iff wrapY).
    peers = (up_ptr, up_rows, down_ptr, down_row0): the launch also forwards
    its boundary output rows into the neighbours' halo rows
    (sg_stencil_launch_p2p; 0 pointers are skipped)."""
    fid, vals = _kind_values(kind)
    d = SgSlabDesc(**desc)
    s = getattr(stream, "cuda_stream", stream)
    if s is None:
        s = _current_stream()
    vptr = vals.ctypes.data_as(C.POINTER(C.c_double)) if vals.size else None
    if peers is None:
        check(_lib.lib().sg_stencil_launch(C.byref(d), ext._c(), fid, vptr, vals.size,
                                           _dtype_code(inp.dtype), C.c_void_p(inp.data_ptr()),
                                           C.c_void_p(out.data_ptr()), C.c_void_p(s or 0)))
        return
    up, up_rows, dn, dn_row0 = peers
    check(_lib.lib().sg_stencil_launch_p2p(C.byref(d), ext._c(), fid, vptr, vals.size, _dtype_code(inp.dtype),
                                           C.c_void_p(inp.data_ptr()), C.c_void_p(out.data_ptr()),
                                           C.c_void_p(up or 0), up_rows, C.c_void_p(dn or 0), dn_row0,
                                           C.c_void_p(s or 0)))
