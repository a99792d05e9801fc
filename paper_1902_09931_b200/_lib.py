"""ctypes binding of the C ABI (include/stengrid/sg.h) in libstengrid_b200.so.

This is the binding a Python caller of the reference-facing boundary would
write. The library is loaded from the package directory
(built in-tree by ``paper_1902_09931_b200.build``); there is no fallback: a
missing library or a missing GPU raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# SG_LIB_PATH overrides the library (A/B experiments with alternative builds).
LIB_PATH = Path(os.environ.get("SG_LIB_PATH") or Path(__file__).resolve().parent / "libstengrid_b200.so")

# sg_status
SG_OK, SG_ERR_INVALID_ARGUMENT, SG_ERR_LOGIC, SG_ERR_PENTA_SOLVE, SG_ERR_DOMAIN, SG_ERR_CUDA, \
    SG_ERR_NO_DEVICE = range(7)

FUNCTIONS = {
    "ch_nonlinear_window": 1,
    "central_difference_window": 2,
    "fn_center": 3,
    "fn_central_second": 4,
    "fn_lap_cube_diff_first": 5,
    "fn_weighted_3x3": 6,
}

# Symbols include/stengrid/sg.h declares (checked by tests/test_capi_symbols.py).
EXPORTED = [
    "sg_abi_version", "sg_last_error", "sg_last_error_system", "sg_launch_count", "sg_init",
    "sg_function_min_coe", "sg_function_name", "sg_wrap", "sg_make_tiles", "sg_plan_create",
    "sg_plan_compute", "sg_plan_swap", "sg_plan_destroy", "sg_plan_sync_to_host",
    "sg_plan_mark_host_dirty", "sg_plan_binding", "sg_plan_valid", "sg_plan_kernel_kind",
    "sg_stencil_launch", "sg_stencil_launch_p2p", "sg_penta_create", "sg_penta_solve", "sg_penta_destroy",
    "sg_ch_default_params", "sg_ch_validate", "sg_ch_create", "sg_ch_step", "sg_ch_set_state",
    "sg_ch_get_field", "sg_ch_device_field", "sg_ch_status", "sg_ch_destroy", "sg_chd_create",
    "sg_chd_geometry", "sg_chd_init", "sg_chd_phase_x", "sg_chd_phase_y", "sg_chd_combine",
    "sg_chd_destroy", "sg_chd_p2p_buffers", "sg_chd_set_peers", "sg_chd_phase_x_p2p", "sg_chd_phase_y_p2p",
    "sg_chd_combine_p2p", "sg_ipc_get_handle", "sg_ipc_open_handle", "sg_ipc_close", "sg_ch_diagnostics", "sg_simpson_mean", "sg_s_metric", "sg_k1_metric", "sg_ch_set_step", "sg_weno_advect",
    "sg_set_device_map", "sg_get_device_map", "sg_plan_workers", "sg_ch_workers", "sg_ch_synchronize",
    "sg_register_function_source", "sg_ch_set_partition",
]


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class LogicError(RuntimeError):
    """std::logic_error in the reference (destroyed plan)."""


class DomainError(ValueError):
    """std::domain_error in the reference."""


class PentaSolveError(RuntimeError):
    """PentaSolveError{system} in the reference (penta.hpp:51-55)."""

    def __init__(self, msg, system):
        super().__init__(msg)
        self.system = system


class CudaError(RuntimeError):
    pass


class NoDeviceError(RuntimeError):
    pass


class SgExtents(C.Structure):
    _fields_ = [("left", C.c_int), ("right", C.c_int), ("top", C.c_int), ("bottom", C.c_int)]


class SgSlabDesc(C.Structure):
    _fields_ = [(n, C.c_int) for n in
                ("nx", "inRows", "inShift", "row0", "row1", "col0", "col1", "wrapX", "wrapY")]


class SgChParams(C.Structure):
    _fields_ = [("D", C.c_double), ("gamma", C.c_double), ("lx", C.c_double), ("ly", C.c_double),
                ("dt", C.c_double), ("T", C.c_double), ("icAmplitude", C.c_double),
                ("nx", C.c_int), ("ny", C.c_int), ("seed", C.c_uint64),
                ("nonlinearEnabled", C.c_int)]


_lib = None


def lib():
    """Load (once) and return the ctypes handle. Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is not built: run `python -m paper_1902_09931_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)
    sig = {
        "sg_abi_version": (C.c_int, []),
        "sg_last_error": (C.c_char_p, []),
        "sg_last_error_system": (C.c_int, []),
        "sg_launch_count": (C.c_uint64, []),
        "sg_init": (C.c_int, [C.c_int]),
        "sg_function_min_coe": (C.c_int, [C.c_int]),
        "sg_function_name": (C.c_char_p, [C.c_int]),
        "sg_register_function_source": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_int)]),
        "sg_ch_set_partition": (C.c_int, [C.c_void_p, C.c_int]),
        "sg_wrap": (C.c_int, [C.c_int64, C.c_int, ip]),
        "sg_make_tiles": (C.c_int, [C.c_int, C.c_int, ip, ip]),
        "sg_plan_create": (C.c_int, [C.c_int, C.c_int, SgExtents, C.c_int, dp, C.c_size_t, C.c_int,
                                     vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(vp)]),
        "sg_plan_compute": (C.c_int, [vp, C.c_int, vp, C.c_int]),
        "sg_plan_swap": (C.c_int, [vp]),
        "sg_plan_destroy": (C.c_int, [C.POINTER(vp)]),
        "sg_plan_sync_to_host": (C.c_int, [vp]),
        "sg_plan_mark_host_dirty": (C.c_int, [vp, C.c_int]),
        "sg_plan_binding": (C.c_int, [vp, C.c_int, C.POINTER(vp), C.POINTER(vp)]),
        "sg_plan_valid": (C.c_int, [vp]),
        "sg_plan_kernel_kind": (C.c_int, [vp]),
        "sg_set_device_map": (C.c_int, [C.c_int]),
        "sg_get_device_map": (C.c_int, []),
        "sg_plan_workers": (C.c_int, [vp, ip, ip, ip, ip, C.c_int]),
        "sg_stencil_launch": (C.c_int, [C.POINTER(SgSlabDesc), SgExtents, C.c_int, dp, C.c_size_t,
                                        C.c_int, vp, vp, vp]),
        "sg_stencil_launch_p2p": (C.c_int, [C.POINTER(SgSlabDesc), SgExtents, C.c_int, dp, C.c_size_t,
                                            C.c_int, vp, vp, vp, C.c_int, vp, C.c_int, vp]),
        "sg_penta_create": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp, C.c_int,
                                      C.POINTER(vp)]),
        "sg_penta_solve": (C.c_int, [vp, vp, C.c_int, vp, C.c_int]),
        "sg_penta_destroy": (C.c_int, [C.POINTER(vp)]),
        "sg_ch_default_params": (None, [C.POINTER(SgChParams)]),
        "sg_ch_validate": (C.c_int, [C.POINTER(SgChParams)]),
        "sg_ch_create": (C.c_int, [C.POINTER(SgChParams), C.c_int, C.c_int, C.POINTER(vp)]),
        "sg_ch_step": (C.c_int, [vp, C.c_int]),
        "sg_ch_set_state": (C.c_int, [vp, vp, vp, C.c_int]),
        "sg_ch_get_field": (C.c_int, [vp, C.c_int, vp, C.c_int]),
        "sg_ch_device_field": (C.c_int, [vp, C.c_int, C.POINTER(vp)]),
        "sg_ch_status": (C.c_int, [vp, ip, dp]),
        "sg_ch_destroy": (C.c_int, [C.POINTER(vp)]),
        "sg_chd_create": (C.c_int, [C.POINTER(SgChParams), C.c_int, C.c_int, C.POINTER(vp)]),
        "sg_chd_geometry": (C.c_int, [vp, ip, ip, ip]),
        "sg_chd_init": (C.c_int, [vp, vp, vp, vp]),
        "sg_chd_phase_x": (C.c_int, [vp, vp, vp, vp, vp]),
        "sg_chd_phase_y": (C.c_int, [vp, vp, vp]),
        "sg_chd_combine": (C.c_int, [vp, vp, vp, vp, vp]),
        "sg_chd_destroy": (C.c_int, [C.POINTER(vp)]),
        "sg_chd_p2p_buffers": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
        "sg_chd_set_peers": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), ip]),
        "sg_chd_phase_x_p2p": (C.c_int, [vp, vp, vp, vp]),
        "sg_chd_phase_y_p2p": (C.c_int, [vp, vp]),
        "sg_chd_combine_p2p": (C.c_int, [vp, vp, vp, vp, vp, vp]),
        "sg_ipc_get_handle": (C.c_int, [vp, vp, C.POINTER(C.c_size_t)]),
        "sg_ipc_open_handle": (C.c_int, [vp, C.POINTER(vp)]),
        "sg_ipc_close": (C.c_int, [vp]),
        "sg_ch_diagnostics": (C.c_int, [vp, dp, dp, dp]),
        "sg_ch_set_step": (C.c_int, [vp, C.c_int]),
        "sg_ch_synchronize": (C.c_int, [vp]),
        "sg_ch_workers": (C.c_int, [vp, ip, ip]),
        "sg_weno_advect": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_double, C.c_double, vp, C.c_int, vp]),
        "sg_simpson_mean": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, dp]),
        "sg_s_metric": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, dp]),
        "sg_k1_metric": (C.c_int, [vp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, dp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(status):
    """Raise the Python twin of the reference's exception for a status."""
    if status == SG_OK:
        return
    L = lib()
    msg = L.sg_last_error().decode()
    if status == SG_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == SG_ERR_LOGIC:
        raise LogicError(msg)
    if status == SG_ERR_PENTA_SOLVE:
        raise PentaSolveError(msg, L.sg_last_error_system())
    if status == SG_ERR_DOMAIN:
        raise DomainError(msg)
    if status == SG_ERR_NO_DEVICE:
        raise NoDeviceError(msg)
    raise CudaError(msg)


def launch_count() -> int:
    return int(lib().sg_launch_count())
