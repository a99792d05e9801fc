"""CSG1 snapshots, diagnostics CSV (the reference's snapshot.cpp formats,
byte for byte) and exact BDF2 checkpoint / resume of a device CHStepper.

CSG1: b"CSG1", <u32 nx, <u32 ny, <f64 dx, <f64 dy, then nx*ny <f64 row-major.
Checkpoint: CSG1(C^n) + CSG1(C^{n-1}) + <u64 step.
"""
from __future__ import annotations

import struct

import numpy as np

from .stencil import Grid2D

MAGIC = b"CSG1"
DIAGNOSTICS_CSV_HEADER = "t,s,k1_inv"


def _write(g: Grid2D, f):
    f.write(MAGIC + struct.pack("<IIdd", g.nx, g.ny, g.dx, g.dy))
    f.write(np.ascontiguousarray(g.values, dtype="<f8").tobytes())


def _read(f) -> Grid2D:
    magic = f.read(4)
    if magic != MAGIC:
        raise RuntimeError("read_snapshot: not a CSG1 file")
    hdr = f.read(24)
    if len(hdr) != 24:
        raise RuntimeError("read_snapshot: truncated file")
    nx, ny, dx, dy = struct.unpack("<IIdd", hdr)
    if nx < 1 or ny < 1 or not dx > 0.0 or not dy > 0.0:
        raise RuntimeError("read_snapshot: invalid header")
    raw = f.read(8 * nx * ny)
    if len(raw) != 8 * nx * ny:
        raise RuntimeError("read_snapshot: truncated file")
    g = Grid2D(nx, ny, dx, dy)
    g.values = np.frombuffer(raw, dtype="<f8").astype(np.float64).reshape(ny, nx).copy()
    return g


def write_snapshot(g: Grid2D, path) -> None:
    """snapshot.cpp:48-66."""
    with open(path, "wb") as f:
        _write(g, f)


def read_snapshot(path) -> Grid2D:
    """snapshot.cpp:68-88."""
    with open(path, "rb") as f:
        return _read(f)


def format_diagnostics_row(d) -> str:
    """snapshot.cpp:92-96 (%.17g)."""
    return "%.17g,%.17g,%.17g" % (d.t, d.s, d.k1Inv)


def write_diagnostics_csv(rows, path) -> None:
    """snapshot.cpp:98-110 (LF endings)."""
    with open(path, "w", newline="\n") as f:
        f.write(DIAGNOSTICS_CSV_HEADER + "\n")
        for d in rows:
            f.write(format_diagnostics_row(d) + "\n")


def save_checkpoint(stepper, path) -> None:
    """Both BDF2 time levels + the step index: exact resume."""
    with open(path, "wb") as f:
        _write(stepper.field(), f)
        _write(stepper.previous_field(), f)
        f.write(struct.pack("<Q", stepper.step_index()))


def load_checkpoint(stepper, path) -> None:
    from . import _lib
    import ctypes as C
    with open(path, "rb") as f:
        curr = _read(f)
        prev = _read(f)
        (step,) = struct.unpack("<Q", f.read(8))
    stepper.set_state(curr, prev)
    _lib.check(_lib.lib().sg_ch_set_step(stepper._h, int(step)))
