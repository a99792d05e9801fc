"""paper_1902_09931_b200 — B200-native cuSten/stengrid stencil engine.

The compute path is libstengrid_b200.so (hand-written sm_100a CUDA behind the
C ABI in include/stengrid/sg.h). This package is the Python host-side mirror
of the reference's API (stengrid/stencil.hpp, penta.hpp, cahn_hilliard.hpp)
plus the multi-GPU y-slab plumbing. There is no CPU fallback.
"""
from . import _lib
from ._lib import (CudaError, DomainError, InvalidArgument, LogicError, NoDeviceError,
                   PentaSolveError, launch_count)
from .stencil import (BoundaryMode, Direction, Extents, FunctionStencil, Grid2D, Residency,
                      StencilPlan, WeightStencil, compute, create_plan, destroy_plan,
                      get_device_map, launch_slab, make_tiles, mark_host_dirty, register_function_source,
                      set_device_map, swap_plan, sync_to_host, wrap)

from .penta import (Axis, PentaBatch, PentaFactor, PeriodicPentaFactor, RhsBatch,
                    build_hyperdiffusion_operator, deinterleave, interleave, solve_batch,
                    solve_periodic_batch)
from .cahn_hilliard import (CHParams, CHStepper, Diagnostics, RunSink, biharmonic_weights, k1_metric,
                            nonlinear_laplacian_coefficients, run, s_metric, simpson_mean)

from .snapshot import (format_diagnostics_row, load_checkpoint, read_snapshot, save_checkpoint,
                       write_diagnostics_csv, write_snapshot)

from .weno import UpwindSide, VelocityField, upwind_side, weno_advect, weno_derivative_7

__all__ = [
    "UpwindSide", "VelocityField", "upwind_side", "weno_advect", "weno_derivative_7",
    "format_diagnostics_row", "load_checkpoint", "read_snapshot", "save_checkpoint",
    "write_diagnostics_csv", "write_snapshot",
    "Axis", "PentaBatch", "PentaFactor", "PeriodicPentaFactor", "RhsBatch",
    "build_hyperdiffusion_operator", "deinterleave", "interleave", "solve_batch",
    "solve_periodic_batch", "CHParams", "CHStepper", "Diagnostics", "biharmonic_weights",
    "nonlinear_laplacian_coefficients", "RunSink", "run", "simpson_mean", "s_metric", "k1_metric",
    "BoundaryMode", "Direction", "Extents", "FunctionStencil", "Grid2D", "Residency",
    "StencilPlan", "WeightStencil", "compute", "create_plan", "destroy_plan", "launch_slab",
    "make_tiles", "mark_host_dirty", "register_function_source", "set_device_map", "get_device_map", "swap_plan", "sync_to_host", "wrap", "InvalidArgument",
    "LogicError", "DomainError", "PentaSolveError", "CudaError", "NoDeviceError", "launch_count",
]
