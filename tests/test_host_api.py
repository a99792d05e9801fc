"""CPU tests of the host-side API mirror (no device calls): parameter
validation, the host setup constants of the CH solver against the golden
fixtures generated from the reference, the penta operator/interleave KATs
and the y-slab geometry. These are the reference's own host-logic tests
(test_cahn_hilliard.cpp, test_penta.cpp, test_grid.cpp) restated."""
import json
import math
from pathlib import Path

import numpy as np
import pytest

import paper_1902_09931_b200 as sg
from paper_1902_09931_b200.slab import Slab

GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "golden.json").read_text())


def _hex(xs):
    return [float.fromhex(x) for x in xs]


def _params(n=64, **kw):
    p = sg.CHParams(nx=n, ny=n)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def test_chparams_defaults_and_validation():
    """cahn_hilliard.hpp:23-39 defaults; cahn_hilliard.cpp:56-66 rules
    (test_cahn_hilliard.cpp:56-75) — host-only, no GPU needed."""
    p = sg.CHParams()
    assert (p.D, p.gamma, p.lx, p.ly, p.seed, p.icAmplitude) == (1.0, 0.01, 2 * math.pi, 2 * math.pi, 1, 0.1)
    _params().validate()
    for field, val in [("nx", 100), ("ny", 96), ("nx", 4), ("dt", 0.0), ("dt", -1.0), ("D", -1.0),
                       ("gamma", 0.0), ("T", 0.0), ("lx", 0.0), ("icAmplitude", -0.1)]:
        with pytest.raises(sg.InvalidArgument):
            _params(**{field: val}).validate()


@pytest.mark.parametrize("n", [64, 1024, 8192])
def test_ch_host_weights_match_reference_golden(n):
    """biharmonic_weights / nonlinear_laplacian_coefficients
    (cahn_hilliard.cpp:78-114) bitwise vs the reference's values."""
    dx = 2 * math.pi / n
    bw = sg.biharmonic_weights(dx, dx)
    nl = sg.nonlinear_laplacian_coefficients(dx, dx)
    want_b = _hex(GOLDEN["kats"][f"biharmonic_weights_{n}"])
    want_n = _hex(GOLDEN["kats"][f"nonlinear_coefficients_{n}"])
    assert [float(x).hex() for x in bw] == [x.hex() for x in want_b]
    assert [float(x).hex() for x in nl] == [x.hex() for x in want_n]
    # the row-major sum is exactly zero (test_cahn_hilliard.cpp:149-158)
    acc = 0.0
    for x in bw:
        acc += x
    assert acc == 0.0


def test_hyperdiffusion_operator_rows_kat():
    """test_penta.cpp:126-159 (penta.cpp:313-335): sigma = 0.25 gives the
    rows {0.25, -1, 2.5, -1, 0.25} in every system; each row sums to 1."""
    for periodic in (False, True):
        m = sg.build_hyperdiffusion_operator(0.25, 8, 3, periodic)
        assert m.periodic == periodic
        for r in (2, 3, 4, 5):
            for b in range(3):
                assert [band[r, b] for band in m.bands()] == [0.25, -1.0, 2.5, -1.0, 0.25]
        assert np.all(m.diag == 2.5)
        if periodic:
            assert np.all(sum(m.bands()) == 1.0)
    with pytest.raises(sg.InvalidArgument):
        sg.build_hyperdiffusion_operator(-1.0, 8, 1, True)


def test_interleave_kat():
    """test_penta.cpp:327-341: a 2 x 3 grid {a b c / d e f} interleaved
    along X is {a d b e c f}; deinterleave inverts it."""
    g = sg.Grid2D(3, 2, 1.0, 1.0)
    g.values[:] = np.array([[1.0, 2.0, 3.0], [4.0, 5.0, 6.0]])
    r = sg.interleave(g, sg.Axis.X)
    assert (r.batchCount, r.n) == (2, 3)
    assert list(r.values.ravel()) == [1.0, 4.0, 2.0, 5.0, 3.0, 6.0]
    back = sg.deinterleave(r, sg.Axis.X, 1.0, 1.0)
    assert np.array_equal(back.values, g.values)
    ry = sg.interleave(g, sg.Axis.Y)
    assert list(ry.values.ravel()) == [1.0, 2.0, 3.0, 4.0, 5.0, 6.0]


@pytest.mark.parametrize("ny,world", [(10, 3), (512, 4), (32768 * 8, 8), (7, 7)])
def test_slab_partition_is_make_tiles(ny, world):
    """The y-slab partition is make_tiles' (grid.cpp:62-82): contiguous,
    ceil-first, covering [0, ny)."""
    tiles = sg.make_tiles(ny, world)
    for r in range(world):
        s = Slab(64, ny, world, r, 1, 1, True)
        assert (s.r0, s.r1) == tiles[r]
        assert s.ext_rows == s.own + 2
        assert s.up == (r - 1) % world and s.down == (r + 1) % world


def test_nonperiodic_slab_keeps_the_frame():
    """Non-periodic outer slabs never write the global frame rows
    (stencil.cpp:35-38)."""
    world, ny = 4, 40
    rows = []
    for r in range(world):
        s = Slab(16, ny, world, r, 2, 1, False)
        a, b = s.output_rows()
        rows += [s.r0 + k for k in range(a, b)]
    assert rows == list(range(2, ny - 1))
    assert Slab(16, ny, world, 0, 2, 1, False).up is None
    assert Slab(16, ny, world, world - 1, 2, 1, False).down is None


def test_weno_host_helpers():
    """weno.hpp:15-17 upwind side and the weno.cpp:33-48 scalar helper."""
    assert sg.upwind_side(-0.0) == sg.UpwindSide.Left
    assert sg.upwind_side(-1e-300) == sg.UpwindSide.Right
    assert sg.upwind_side(2.0) == sg.UpwindSide.Left
    # a linear profile has the exact derivative on both sides
    w7 = [0.5 * k for k in range(7)]
    for side in (sg.UpwindSide.Left, sg.UpwindSide.Right):
        d = sg.weno_derivative_7(w7, 10.0, side)
        assert abs(abs(d) - 5.0) < 1e-12
