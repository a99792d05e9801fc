"""GPU: WENO5 advection (tests/test_weno.cpp restated) — bitwise vs the
reference library, plus the reference's analytic checks."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def fields(sg, nx, ny, seed):
    rng = np.random.default_rng(seed)
    dx, dy = 2 * math.pi / nx, 2 * math.pi / ny
    phi = sg.Grid2D.from_array(rng.uniform(-1, 1, (ny, nx)), dx, dy)
    u = sg.Grid2D.from_array(rng.uniform(-1, 1, (ny, nx)), dx, dy)
    v = sg.Grid2D.from_array(rng.uniform(-1, 1, (ny, nx)), dx, dy)
    return phi, sg.VelocityField(u, v)


@pytest.mark.parametrize("nx,ny", [(7, 7), (64, 48), (129, 70), (512, 256)])
def test_weno_bitwise_vs_reference(sg, ref, nx, ny):
    phi, vel = fields(sg, nx, ny, nx * 3 + ny)
    got = sg.weno_advect(phi, vel).values
    want = ref.weno_advect(phi.values, vel.u.values, vel.v.values, phi.dx, phi.dy, tiles=2, workers=2)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_weno_constant_and_sine(sg):
    n = 128
    dx = 2 * math.pi / n
    x = np.arange(n) * dx
    const = sg.Grid2D.from_array(np.full((n, n), 0.7), dx, dx)
    one = sg.Grid2D.from_array(np.ones((n, n)), dx, dx)
    vel = sg.VelocityField(one, one)
    assert np.all(sg.weno_advect(const, vel).values == 0.0)
    phi = sg.Grid2D.from_array(np.tile(np.sin(x), (n, 1)), dx, dx)
    out = sg.weno_advect(phi, sg.VelocityField(one, sg.Grid2D.from_array(np.zeros((n, n)), dx, dx))).values
    assert np.max(np.abs(out + np.cos(x)[None, :])) < 1e-6  # -u dphi/dx with u = 1


def test_weno_validation(sg):
    phi, vel = fields(sg, 6, 8, 1)
    with pytest.raises(sg.InvalidArgument):
        sg.weno_advect(phi, vel)
    phi, vel = fields(sg, 8, 8, 1)
    vel.u = sg.Grid2D(9, 8)
    with pytest.raises(sg.InvalidArgument):
        sg.weno_advect(phi, vel)


def test_weno_scalar_helper_matches_reference_formula(sg):
    w7 = [0.1, 0.3, -0.2, 0.5, 0.7, 0.2, -0.4]
    left = sg.weno_derivative_7(w7, 10.0, sg.UpwindSide.Left)
    right = sg.weno_derivative_7(w7, 10.0, sg.UpwindSide.Right)
    assert math.isfinite(left) and math.isfinite(right) and left != right
    assert sg.upwind_side(-0.0) == sg.UpwindSide.Left and sg.upwind_side(-1e-300) == sg.UpwindSide.Right
