"""oracle/oracle.py — ctypes front-end to the CPU CHECKERS. TEST INFRASTRUCTURE.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline — never as the product path.

Two libraries are wrapped:

* ``Restatement`` → ``oracle/liboracle.so``: the plain-C restatement of the
  reference hot path (``stengrid_oracle.c``; every function cites the
  reference file:line it follows).
* ``Reference`` → ``oracle/_ref/libstengrid_ref.so``: the UNMODIFIED
  reference library compiled from ``/root/reference/proj/src`` by
  ``oracle/Makefile`` (with ``ref_driver.cpp`` as the extern "C" shim).

Both take/return numpy float64 arrays in the reference's row-major layout
(entry (i, j) at ``j*nx + i``, ``grid.hpp:11-49``).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
RESTATEMENT_SO = HERE / "liboracle.so"
REFERENCE_SO = HERE / "_ref" / "libstengrid_ref.so"

# Function-stencil ids, shared with include/stengrid/sg.h (SG_FN_*).
FN_IDS = {
    "weights": 0,
    "ch_nonlinear_window": 1,
    "central_difference_window": 2,
    "fn_center": 3,
    "fn_central_second": 4,
    "fn_lap_cube_diff_first": 5,
    "fn_weighted_3x3": 6,
}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def _d(a):
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, code, msg, system=-1):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.system = system


def build():
    """Compile both checkers (make -C oracle). The reference half is skipped
    when /root/reference is absent (the GPU box), keeping any prebuilt .so."""
    import subprocess

    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


class Restatement:
    def __init__(self, path=RESTATEMENT_SO):
        if not Path(path).exists():
            build()
        L = self.lib = C.CDLL(str(path))
        L.orc_wrap.restype = C.c_int
        L.orc_wrap.argtypes = [C.c_longlong, C.c_int]
        L.orc_make_tiles.argtypes = [C.c_int, C.c_int, _ip, _ip]
        L.orc_stencil.argtypes = [C.c_int, _ip, C.c_int, _dp, _dp, _dp, C.c_int, C.c_int]
        L.orc_penta_solve.argtypes = [C.c_int, C.c_int, C.c_int] + [_dp] * 6
        L.orc_hyperdiffusion_operator.argtypes = [C.c_double, C.c_int, C.c_int, C.c_int] + [_dp] * 5
        L.orc_ch_initial_condition.argtypes = [C.c_uint64, C.c_double, C.c_longlong, _dp]
        L.orc_ch_weights.argtypes = [C.c_double, C.c_double, _dp, _dp]
        L.orc_ch_run.argtypes = [_dp, _ip, C.c_int, _dp, _dp]
        L.orc_uniform_factor_tables.argtypes = [C.c_double, C.c_int] + [_dp] * 6 + [_dp, _ip, _dp]

    def wrap(self, i, n):
        return self.lib.orc_wrap(i, n)

    def make_tiles(self, ny, num_tiles):
        b = (C.c_int * num_tiles)()
        e = (C.c_int * num_tiles)()
        if self.lib.orc_make_tiles(ny, num_tiles, b, e) != 0:
            raise ValueError("make_tiles: invalid arguments")
        return [(b[k], e[k]) for k in range(num_tiles)]

    def stencil(self, inp, ext, weights, *, periodic=True, fn="weights", out=None):
        """One application. ``inp`` is (ny, nx); ``out`` (same shape) supplies
        the untouched frame for non-periodic stencils (zeros if omitted)."""
        inp = _f64(inp)
        ny, nx = inp.shape
        res = np.zeros_like(inp) if out is None else _f64(out).copy()
        e = (C.c_int * 4)(*ext)
        w = _f64(weights) if len(weights) else np.zeros(1)
        rc = self.lib.orc_stencil(int(periodic), e, FN_IDS[fn], _d(w), _d(inp), _d(res), nx, ny)
        if rc != 0:
            raise ValueError("unknown function id")
        return res

    def penta_solve(self, periodic, bands, rhs):
        """bands = (e, c, d, a, b) each (n, B) interleaved; rhs (n, B)."""
        e, c, d, a, b = (_f64(x) for x in bands)
        n, B = rhs.shape
        y = _f64(rhs).copy()
        bad = self.lib.orc_penta_solve(int(periodic), B, n, _d(e), _d(c), _d(d), _d(a), _d(b), _d(y))
        if bad >= 0:
            raise OracleError(3, "penta: zero pivot / singular capacitance", bad)
        return y

    def hyperdiffusion_operator(self, sigma, n, B, periodic):
        out = [np.empty((n, B)) for _ in range(5)]
        self.lib.orc_hyperdiffusion_operator(sigma, n, B, int(periodic), *(_d(x) for x in out))
        return tuple(out)

    def ch_initial_condition(self, nx, ny, seed=1, amp=0.1):
        out = np.empty((ny, nx))
        self.lib.orc_ch_initial_condition(seed, amp, nx * ny, _d(out))
        return out

    def ch_weights(self, dx, dy):
        w = np.empty(25)
        n = np.empty(9)
        self.lib.orc_ch_weights(dx, dy, _d(w), _d(n))
        return w, n

    def ch_run(self, params, steps, curr, prev):
        dp = np.array([params["D"], params["gamma"], params["lx"], params["ly"], params["dt"]])
        ip = (C.c_int * 3)(params["nx"], params["ny"], int(params.get("nonlinear", True)))
        c = _f64(curr).copy()
        p = _f64(prev).copy()
        bad = self.lib.orc_ch_run(_d(dp), ip, steps, _d(c), _d(p))
        if bad >= 0:
            raise OracleError(3, "penta factor failed", bad)
        return c, p

    def uniform_factor_tables(self, sigma, n):
        m1, m2, dInv, ap, bp = (np.empty(n) for _ in range(5))
        W = np.empty((4, n))
        K = np.empty(16)
        piv = (C.c_int * 4)()
        cw = np.empty(6)
        bad = self.lib.orc_uniform_factor_tables(sigma, n, _d(m1), _d(m2), _d(dInv), _d(ap), _d(bp),
                                                 _d(W), _d(K), piv, _d(cw))
        return dict(m1=m1, m2=m2, dInv=dInv, ap=ap, bp=bp, W=W, K=K, piv=list(piv), cw=cw, bad=bad)


class Reference:
    """The real reference library (oracle/_ref). Raises FileNotFoundError if
    it was never built (e.g. /root/reference absent and no prebuilt .so)."""

    def __init__(self, path=REFERENCE_SO):
        if not Path(path).exists():
            raise FileNotFoundError(f"{path} not built (run make -C oracle where /root/reference exists)")
        L = self.lib = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_error.argtypes = [_ip]
        L.ref_wrap.argtypes = [C.c_longlong, C.c_int, _ip]
        L.ref_make_tiles.argtypes = [C.c_int, C.c_int, _ip, _ip]
        L.ref_stencil.argtypes = [C.c_int, C.c_int, _ip, C.c_int, _dp, C.c_int, _dp, _dp,
                                  C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_stencil_timed.argtypes = [C.c_int, C.c_int, _ip, C.c_int, _dp, C.c_int, _dp,
                                        C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.ref_apply_at.argtypes = [C.c_int, _ip, C.c_int, _dp, C.c_int, _dp, C.c_int, C.c_int,
                                   C.c_int, C.c_int, _dp]
        L.ref_penta_solve.argtypes = [C.c_int, C.c_int, C.c_int] + [_dp] * 6 + [C.c_int]
        L.ref_hyperdiffusion_operator.argtypes = [C.c_double, C.c_int, C.c_int, C.c_int] + [_dp] * 5
        L.ref_ch_weights.argtypes = [C.c_double, C.c_double, _dp, _dp]
        L.ref_ch_initial_condition.argtypes = [_dp, C.POINTER(C.c_longlong), _dp]
        L.ref_ch_run.argtypes = [_dp, C.POINTER(C.c_longlong), C.c_int, C.c_int, C.c_int, C.c_int,
                                 _dp, _dp]
        L.ref_ch_timed.argtypes = [_dp, C.POINTER(C.c_longlong), C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.ref_ch_diagnostics.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_double, _dp, _dp]
        L.ref_write_snapshot.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_char_p]
        L.ref_read_snapshot.argtypes = [C.c_char_p, _ip, _ip, _dp, _dp, _dp, C.c_longlong]
        L.ref_write_diagnostics_csv.argtypes = [_dp, C.c_int, C.c_char_p]
        L.ref_weno_advect.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, _dp]

    def _check(self, rc):
        if rc != 0:
            sysidx = C.c_int(-1)
            msg = self.lib.ref_last_error(C.byref(sysidx)).decode()
            raise OracleError(rc, msg, sysidx.value)

    def wrap(self, i, n):
        out = C.c_int()
        self._check(self.lib.ref_wrap(i, n, C.byref(out)))
        return out.value

    def make_tiles(self, ny, num_tiles):
        b = (C.c_int * max(num_tiles, 1))()
        e = (C.c_int * max(num_tiles, 1))()
        self._check(self.lib.ref_make_tiles(ny, num_tiles, b, e))
        return [(b[k], e[k]) for k in range(num_tiles)]

    def stencil(self, inp, ext, weights, *, direction=2, periodic=True, fn="weights", out=None,
                tiles=1, workers=1, applications=1):
        inp = _f64(inp)
        ny, nx = inp.shape
        res = np.zeros_like(inp) if out is None else _f64(out).copy()
        e = (C.c_int * 4)(*ext)
        w = _f64(weights) if len(weights) else np.zeros(1)
        self._check(self.lib.ref_stencil(direction, int(periodic), e, FN_IDS[fn], _d(w), len(weights),
                                         _d(inp), _d(res), nx, ny, tiles, workers, applications))
        return res

    def stencil_timed(self, inp, ext, weights, *, direction=2, periodic=True, fn="weights",
                      tiles=1, workers=1, warmup=1, reps=1):
        """Seconds PER compute() of the reference (mean over `reps`)."""
        inp = _f64(inp)
        ny, nx = inp.shape
        e = (C.c_int * 4)(*ext)
        w = _f64(weights)
        secs = C.c_double()
        self._check(self.lib.ref_stencil_timed(direction, int(periodic), e, FN_IDS[fn], _d(w),
                                               len(weights), _d(inp), nx, ny, tiles, workers,
                                               warmup, reps, C.byref(secs)))
        return secs.value

    def apply_at(self, inp, ext, weights, i, j, *, periodic=True, fn="weights"):
        inp = _f64(inp)
        ny, nx = inp.shape
        e = (C.c_int * 4)(*ext)
        w = _f64(weights) if len(weights) else np.zeros(1)
        out = C.c_double()
        self._check(self.lib.ref_apply_at(int(periodic), e, FN_IDS[fn], _d(w), len(weights), _d(inp),
                                          nx, ny, i, j, C.byref(out)))
        return out.value

    def penta_solve(self, periodic, bands, rhs, workers=1):
        e, c, d, a, b = (_f64(x) for x in bands)
        n, B = rhs.shape
        y = _f64(rhs).copy()
        self._check(self.lib.ref_penta_solve(int(periodic), B, n, _d(e), _d(c), _d(d), _d(a), _d(b),
                                             _d(y), workers))
        return y

    def hyperdiffusion_operator(self, sigma, n, B, periodic):
        out = [np.empty((n, B)) for _ in range(5)]
        self._check(self.lib.ref_hyperdiffusion_operator(sigma, n, B, int(periodic),
                                                         *(_d(x) for x in out)))
        return tuple(out)

    def ch_weights(self, dx, dy):
        w = np.empty(25)
        n = np.empty(9)
        self._check(self.lib.ref_ch_weights(dx, dy, _d(w), _d(n)))
        return w, n

    @staticmethod
    def _ch_params(p):
        dp = np.array([p["D"], p["gamma"], p["lx"], p["ly"], p["dt"], p.get("T", 1.0),
                       p.get("amp", 0.1)])
        ip = (C.c_longlong * 4)(p["nx"], p["ny"], p.get("seed", 1), int(p.get("nonlinear", True)))
        return dp, ip

    def ch_initial_condition(self, p):
        dp, ip = self._ch_params(p)
        out = np.empty((p["ny"], p["nx"]))
        self._check(self.lib.ref_ch_initial_condition(_d(dp), ip, _d(out)))
        return out

    def ch_run(self, p, steps, curr=None, prev=None, tiles=1, workers=1):
        dp, ip = self._ch_params(p)
        set_state = curr is not None
        c = _f64(curr).copy() if set_state else np.empty((p["ny"], p["nx"]))
        pr = _f64(prev).copy() if set_state else np.empty((p["ny"], p["nx"]))
        self._check(self.lib.ref_ch_run(_d(dp), ip, tiles, workers, steps, int(set_state), _d(c), _d(pr)))
        return c, pr

    def ch_timed(self, p, steps, warmup=1, tiles=1, workers=1):
        """Seconds PER STEP of the reference CHStepper::step over `steps`
        timed steps (after `warmup`)."""
        dp, ip = self._ch_params(p)
        secs = C.c_double()
        self._check(self.lib.ref_ch_timed(_d(dp), ip, tiles, workers, warmup, steps, C.byref(secs)))
        return secs.value

    def write_snapshot(self, values, dx, dy, path):
        v = _f64(values)
        ny, nx = v.shape
        self._check(self.lib.ref_write_snapshot(_d(v), nx, ny, dx, dy, str(path).encode()))

    def read_snapshot(self, path, cap=1 << 22):
        nx, ny = C.c_int(), C.c_int()
        dx, dy = C.c_double(), C.c_double()
        buf = np.empty(cap)
        self._check(self.lib.ref_read_snapshot(str(path).encode(), C.byref(nx), C.byref(ny), C.byref(dx),
                                               C.byref(dy), _d(buf), cap))
        return buf[: nx.value * ny.value].reshape(ny.value, nx.value).copy(), dx.value, dy.value

    def weno_advect(self, phi, u, v, dx, dy, tiles=1, workers=1):
        phi, u, v = _f64(phi), _f64(u), _f64(v)
        ny, nx = phi.shape
        out = np.empty_like(phi)
        self._check(self.lib.ref_weno_advect(_d(phi), _d(u), _d(v), nx, ny, dx, dy, tiles, workers, _d(out)))
        return out

    def write_diagnostics_csv(self, rows, path):
        r = _f64(np.asarray(rows, dtype=np.float64).reshape(-1, 3))
        self._check(self.lib.ref_write_diagnostics_csv(_d(r), r.shape[0], str(path).encode()))

    def ch_diagnostics(self, field, dx, dy):
        f = _f64(field)
        ny, nx = f.shape
        s = C.c_double()
        k = C.c_double()
        self._check(self.lib.ref_ch_diagnostics(_d(f), nx, ny, dx, dy, C.byref(s), C.byref(k)))
        return s.value, k.value


def ch_params(n=64, ny=None, dt_factor=0.1, **kw):
    """CHParams defaults (cahn_hilliard.hpp:23-39) with dt = dt_factor*dx."""
    ny = n if ny is None else ny
    lx = ly = 2.0 * np.pi
    p = dict(D=1.0, gamma=0.01, nx=n, ny=ny, lx=lx, ly=ly, T=1.0, seed=1, amp=0.1, nonlinear=True)
    p["dt"] = dt_factor * (lx / n)
    p.update(kw)
    return p
