"""GPU parity tests for the stencil engine (run on the B200: ``pytest -m gpu``).

Restates the reference's stencil tests (tests/test_stencil.cpp,
tests/acceptance.cpp criterion 2) against the sm_100a path, with the C
restatement (oracle/liboracle.so, pinned bitwise to the reference in
tests/test_oracle.py) as the checker. FP64 parity is BITWISE (0 ulp);
FP32 is within 1e-5 relative of the FP64 oracle on float-rounded inputs
(BASELINE.json north_star tolerance).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TWO_PI = 2.0 * math.pi
FAST_WEIGHT_EXTENTS = [(l, t) for t in range(5) for l in range(5)]


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def run_gpu(sg, inp, ext, weights, *, direction=2, periodic=True, fn=None, out=None, tiles=1,
            workers=1, applications=1, expect_kind=None):
    """create_plan / compute (/ swap / compute ...) through the Python mirror
    of the reference API with HOST grids (the reference's own usage)."""
    ny, nx = inp.shape
    gi = sg.Grid2D.from_array(inp.copy())
    go = sg.Grid2D.from_array(np.zeros_like(inp) if out is None else out.copy())
    e = sg.Extents(*ext)
    kind = sg.WeightStencil(e, list(weights)) if fn is None else sg.FunctionStencil(e, fn, list(weights))
    plan = sg.create_plan(direction, sg.BoundaryMode.Periodic if periodic else sg.BoundaryMode.NonPeriodic,
                          kind, gi, go, tiles, workers)
    if expect_kind is not None:
        assert plan.kernel_kind() == expect_kind
    for a in range(applications):
        sg.compute(plan)
        if a + 1 < applications:
            sg.swap_plan(plan)
    res = plan.output().values.copy()
    sg.destroy_plan(plan)
    return res


def direction_of(ext):
    l, r, t, b = ext
    if t == 0 and b == 0:
        return 0
    if l == 0 and r == 0:
        return 1
    return 2


# ---------------------------------------------------------------- acceptance


def test_acceptance_criterion_2_random_periodic_bitwise(sg, orc):
    """acceptance.cpp:104-151 — 200 random periodic cases, nx, ny in [1,9],
    extents <= min(2, n-1), bitwise vs brute force."""
    rng = np.random.default_rng(99)
    mismatches = 0
    for _ in range(200):
        nx, ny = (int(v) for v in rng.integers(1, 10, 2))
        d = int(rng.integers(0, 3))
        e = [0, 0, 0, 0]
        if d != 1:
            e[0], e[1] = (int(v) for v in rng.integers(0, min(2, nx - 1) + 1, 2))
        if d != 0:
            e[2], e[3] = (int(v) for v in rng.integers(0, min(2, ny - 1) + 1, 2))
        W = (e[0] + e[1] + 1) * (e[2] + e[3] + 1)
        inp = rng.uniform(-2, 2, (ny, nx))
        w = rng.uniform(-2, 2, W)
        got = run_gpu(sg, inp, e, w, direction=d)
        want = orc.stencil(inp, e, w)
        mismatches += int((got.view(np.uint64) != want.view(np.uint64)).sum())
    assert mismatches == 0


# ------------------------------------------------------- fast-path coverage


@pytest.mark.parametrize("l,t", FAST_WEIGHT_EXTENTS)
@pytest.mark.parametrize("periodic", [True, False])
def test_strip_kernel_weights_bitwise(sg, orc, l, t, periodic):
    rng = np.random.default_rng(1000 + 10 * l + t)
    nx, ny = 320, 97  # 5 FP64 strips, odd row count
    ext = (l, l, t, t)
    inp = rng.uniform(-1, 1, (ny, nx))
    w = rng.uniform(-2, 2, (2 * l + 1) * (2 * t + 1))
    sentinel = np.full_like(inp, -12345.678)
    got = run_gpu(sg, inp, ext, w, direction=direction_of(ext), periodic=periodic, out=sentinel,
                  expect_kind=1)
    want = orc.stencil(inp, ext, w, periodic=periodic, out=sentinel)
    assert bits_equal(got, want)


@pytest.mark.parametrize("nx", [2, 4, 6, 62, 64, 66, 130, 192])
def test_strip_kernel_partial_strips_and_narrow_grids(sg, orc, nx):
    """Partial last strip, grids narrower than one strip, windows touching
    wrapped columns from both sides."""
    rng = np.random.default_rng(nx)
    ny = 23
    for l in (1, 2):
        if l >= nx:
            continue
        ext = (l, l, 1, 1)
        inp = rng.uniform(-1, 1, (ny, nx))
        w = rng.uniform(-2, 2, (2 * l + 1) * 3)
        for periodic in (True, False):
            got = run_gpu(sg, inp, ext, w, periodic=periodic, expect_kind=1)
            want = orc.stencil(inp, ext, w, periodic=periodic)
            assert bits_equal(got, want), (nx, l, periodic)


FUNCS = [
    ("ch_nonlinear_window", (1, 1, 1, 1), 9),
    ("fn_weighted_3x3", (1, 1, 1, 1), 9),
    ("fn_center", (1, 1, 1, 1), 0),
    ("fn_lap_cube_diff_first", (1, 1, 1, 1), 2),
    ("fn_central_second", (1, 1, 0, 0), 1),
    ("central_difference_window", (1, 1, 0, 0), 1),
]


@pytest.mark.parametrize("fn,ext,ncoe", FUNCS)
@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("shape", [(64, 40), (37, 11)])  # fast path / generic path
def test_function_stencils_bitwise(sg, orc, fn, ext, ncoe, periodic, shape):
    nx, ny = shape
    rng = np.random.default_rng(hash((fn, nx)) & 0xFFFF)
    inp = rng.uniform(-1.5, 1.5, (ny, nx))
    coe = rng.uniform(-2, 2, max(ncoe, 1))[:ncoe]
    got = run_gpu(sg, inp, ext, coe, direction=direction_of(ext), periodic=periodic, fn=fn,
                  expect_kind=1 if nx % 2 == 0 else 2)
    want = orc.stencil(inp, ext, coe, periodic=periodic, fn=fn)
    assert bits_equal(got, want)


def test_function_stencil_generic_shapes(sg, orc):
    """Device functions on windows wider than their natural shape run on the
    generic kernel (fn_center on a 5x5 window reads w[rs+1])."""
    rng = np.random.default_rng(5)
    inp = rng.uniform(-1, 1, (19, 26))
    got = run_gpu(sg, inp, (2, 2, 2, 2), [], fn="fn_center", expect_kind=0)
    want = orc.stencil(inp, (2, 2, 2, 2), [], fn="fn_center")
    assert bits_equal(got, want)


def test_asymmetric_and_large_extents_generic(sg, orc):
    """test_stencil.cpp:557-568 (asymmetric {3,1,0,0}) and windows beyond the
    fast-path set, incl. > 256 weights (device weight buffer)."""
    rng = np.random.default_rng(161)
    for ext, shape in [((3, 1, 0, 0), (9, 13)), ((2, 1, 1, 2), (18, 24)), ((6, 6, 0, 0), (5, 40)),
                       ((10, 9, 7, 8), (30, 31))]:
        ny, nx = shape
        inp = rng.uniform(-1, 1, (ny, nx))
        W = (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
        w = rng.uniform(-2, 2, W)
        for periodic in (True, False):
            got = run_gpu(sg, inp, ext, w, direction=direction_of(ext), periodic=periodic)
            want = orc.stencil(inp, ext, w, periodic=periodic)
            assert bits_equal(got, want), ext


# ----------------------------------------------------- restated unit tests


def test_identity_stencil_bitwise_all_directions_modes(sg):
    """test_stencil.cpp:278-289."""
    rng = np.random.default_rng(51)
    inp = rng.uniform(-1, 1, (11, 9))
    for d in (0, 1, 2):
        for periodic in (True, False):
            got = run_gpu(sg, inp, (0, 0, 0, 0), [1.0], direction=d, periodic=periodic, tiles=2,
                          workers=2)
            assert bits_equal(got, inp)


def test_cross_derivative_exact_on_i2j2(sg):
    """test_stencil.cpp:291-303 — d4/(dx2 dy2) of i^2 j^2 is exactly 4."""
    i = np.arange(8, dtype=np.float64)
    g = (i[None, :] ** 2) * (i[:, None] ** 2)
    got = run_gpu(sg, g, (1, 1, 1, 1), [1, -2, 1, -2, 4, -2, 1, -2, 1], periodic=False)
    assert np.all(got[1:7, 1:7] == 4.0)


def test_periodic_second_derivative_of_sine(sg):
    """test_stencil.cpp:263-276."""
    n = 1024
    dx = TWO_PI / n
    x = np.sin(np.arange(n) * dx)[None, :]
    c = 1.0 / (dx * dx)
    got = run_gpu(sg, x, (1, 1, 0, 0), [c, -2 * c, c], direction=0)
    err = np.max(np.abs(got[0] + np.sin(np.arange(n) * dx)))
    assert 1e-6 < err < 5e-6


def second_derivative_max_error(sg, n, coeffs, hw):
    dx = TWO_PI / n
    x = np.sin(np.arange(n) * dx)[None, :]
    s = 1.0 / (dx * dx)
    got = run_gpu(sg, x, (hw, hw, 0, 0), [c * s for c in coeffs], direction=0)
    return np.max(np.abs(got[0] + np.sin(np.arange(n) * dx)))


def test_convergence_orders(sg):
    """test_stencil.cpp:489-501 / acceptance criterion 1."""
    r2 = second_derivative_max_error(sg, 128, [1, -2, 1], 1) / second_derivative_max_error(sg, 256, [1, -2, 1], 1)
    c8 = [-1 / 560, 8 / 315, -1 / 5, 8 / 5, -205 / 72, 8 / 5, -1 / 5, 8 / 315, -1 / 560]
    r8 = second_derivative_max_error(sg, 32, c8, 4) / second_derivative_max_error(sg, 64, c8, 4)
    assert 3.6 < r2 < 4.4
    assert 256 * 0.8 < r8 < 256 * 1.2


def test_weights_and_function_bitwise_equivalent(sg):
    """test_stencil.cpp:345-362, 374-388."""
    rng = np.random.default_rng(101)
    inp = rng.uniform(-1, 1, (6, 9))
    w = rng.uniform(-2, 2, 9)
    for periodic in (True, False):
        a = run_gpu(sg, inp, (1, 1, 1, 1), w, periodic=periodic, tiles=3, workers=2)
        b = run_gpu(sg, inp, (1, 1, 1, 1), w, periodic=periodic, fn="fn_weighted_3x3", tiles=3, workers=2)
        assert bits_equal(a, b)
    dx = TWO_PI / 32
    c = 1.0 / (dx * dx)
    inp = rng.uniform(-1, 1, (4, 32))
    a = run_gpu(sg, inp, (1, 1, 0, 0), [c, -2 * c, c], direction=0, tiles=2, workers=2)
    b = run_gpu(sg, inp, (1, 1, 0, 0), [c], direction=0, fn="fn_central_second", tiles=2, workers=2)
    assert bits_equal(a, b)


def test_tile_and_worker_invariance(sg, orc):
    """test_stencil.cpp:390-409."""
    rng = np.random.default_rng(111)
    inp = rng.uniform(-1, 1, (13, 16))
    w = rng.uniform(-2, 2, 15)
    ref = orc.stencil(inp, (2, 2, 1, 1), w)
    for tiles in (1, 2, 3, 5, 13):
        for workers in (1, 2, 4):
            assert bits_equal(run_gpu(sg, inp, (2, 2, 1, 1), w, tiles=tiles, workers=workers), ref)


def test_nonperiodic_leaves_exactly_the_frame(sg):
    """test_stencil.cpp:411-440 — sentinel -12345.678 survives in the frame only."""
    sentinel = -12345.678
    rng = np.random.default_rng(121)
    for d, ext in [(0, (2, 3, 0, 0)), (1, (0, 0, 1, 2)), (2, (1, 2, 2, 1))]:
        inp = rng.uniform(-1, 1, (9, 11))
        W = (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
        out = run_gpu(sg, inp, ext, rng.uniform(-2, 2, W), direction=d, periodic=False,
                      out=np.full_like(inp, sentinel), tiles=3, workers=2)
        jj, ii = np.mgrid[0:9, 0:11]
        frame = (ii < ext[0]) | (ii >= 11 - ext[1]) | (jj < ext[2]) | (jj >= 9 - ext[3])
        assert np.all(out[frame] == sentinel)
        assert np.all(out[~frame] != sentinel)


def test_cyclic_shift_equivariance(sg):
    """test_stencil.cpp:442-460."""
    rng = np.random.default_rng(131)
    inp = rng.uniform(-1, 1, (10, 12))
    w = rng.uniform(-2, 2, 9)
    plain = run_gpu(sg, inp, (1, 1, 1, 1), w, tiles=2, workers=2)
    for si, sj in [(3, 2), (-5, 7), (1, 0)]:
        shifted = np.roll(inp, (sj, si), axis=(0, 1))
        got = run_gpu(sg, shifted, (1, 1, 1, 1), w, tiles=2, workers=2)
        assert bits_equal(got, np.roll(plain, (sj, si), axis=(0, 1)))


def test_linearity(sg):
    """test_stencil.cpp:462-487 — 1e-13 relative."""
    rng = np.random.default_rng(141)
    f = rng.uniform(-1, 1, (8, 10))
    g = rng.uniform(-1, 1, (8, 10))
    w = rng.uniform(-2, 2, 9)
    combo = 1.7 * f + -0.3 * g
    oc = run_gpu(sg, combo, (1, 1, 1, 1), w)
    want = 1.7 * run_gpu(sg, f, (1, 1, 1, 1), w) + -0.3 * run_gpu(sg, g, (1, 1, 1, 1), w)
    assert np.allclose(oc, want, rtol=1e-13, atol=1e-13 * np.abs(want).max())


def test_compute_swap_compute(sg, orc):
    """test_stencil.cpp:227-249 — the second pass lands back in `in`."""
    rng = np.random.default_rng(31)
    inp = rng.uniform(-1, 1, (9, 14))
    w = [0.5, -1.0, 0.5]
    gi = sg.Grid2D.from_array(inp.copy())
    go = sg.Grid2D(14, 9)
    plan = sg.create_plan(sg.Direction.X, sg.BoundaryMode.Periodic, sg.WeightStencil(sg.Extents(1, 1), w),
                          gi, go, 3, 2)
    sg.compute(plan)
    sg.swap_plan(plan)
    sg.compute(plan)
    ref2 = orc.stencil(orc.stencil(inp, (1, 1, 0, 0), w), (1, 1, 0, 0), w)
    assert bits_equal(gi.values, ref2)


def test_swap_semantics_and_lifecycle(sg):
    """test_stencil.cpp:123-261 — lifecycle, swap, destroy idempotence, errors."""
    a = sg.Grid2D.from_array(np.random.default_rng(21).uniform(-1, 1, (6, 10)))
    b = sg.Grid2D(10, 6)
    acopy = a.values.copy()
    plan = sg.create_plan(sg.Direction.X, sg.BoundaryMode.Periodic,
                          sg.WeightStencil(sg.Extents(1, 1), [0.25, 0.5, 0.25]), a, b, 1, 1)
    assert plan.input() is a and plan.output() is b
    sg.swap_plan(plan)
    assert plan.input() is b and plan.output() is a
    sg.swap_plan(plan)
    sg.compute(plan)
    sg.destroy_plan(plan)
    assert not plan.valid()
    sg.destroy_plan(plan)
    with pytest.raises(sg.LogicError):
        sg.compute(plan)
    with pytest.raises(sg.LogicError):
        sg.swap_plan(plan)
    assert bits_equal(a.values, acopy)


def test_create_plan_rejects_invalid_setups(sg):
    """test_stencil.cpp:134-183 — every case raises std::invalid_argument."""
    a, b, small = sg.Grid2D(16, 8), sg.Grid2D(16, 8), sg.Grid2D(4, 8)
    X, Y, P = sg.Direction.X, sg.Direction.Y, sg.BoundaryMode.Periodic
    W, F, E = sg.WeightStencil, sg.FunctionStencil, sg.Extents
    w3 = [1.0, -2.0, 1.0]
    cases = [
        (X, W(E(1, 1), w3), a, a, 1),
        (X, W(E(16, 0), [1.0] * 17), a, b, 1),
        (X, W(E(1, 1), []), a, b, 1),
        (X, W(E(1, 1), [1.0, 2.0]), a, b, 1),
        (X, W(E(1, 1), [1.0, float("nan"), 1.0]), a, b, 1),
        (X, W(E(1, 1, 1, 0), [1.0] * 6), a, b, 1),
        (Y, W(E(1, 0, 1, 1), [1.0] * 6), a, b, 1),
        (X, W(E(1, 1), w3), a, small, 1),
        (X, F(E(1, 1), None, []), a, b, 1),
        (X, W(E(1, 1), w3), a, b, 9),
    ]
    for d, kind, gi, go, tiles in cases:
        with pytest.raises(sg.InvalidArgument):
            sg.create_plan(d, P, kind, gi, go, tiles, 1)
    with pytest.raises(sg.InvalidArgument):
        sg.create_plan(X, P, W(E(1, 1), w3), a, b, 1, 0)


def test_residency_hint_does_not_change_results(sg):
    """test_stencil.cpp:515-525 + device residency round trip."""
    rng = np.random.default_rng(151)
    inp = rng.uniform(-1, 1, (8, 8))
    w = rng.uniform(-2, 2, 9)
    gi = sg.Grid2D.from_array(inp)
    oh, od = sg.Grid2D(8, 8), sg.Grid2D(8, 8)
    kind = sg.WeightStencil(sg.Extents(1, 1, 1, 1), list(w))
    ph = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, kind, gi, oh, 1, 1)
    pd = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, kind, gi, od, 1, 1)
    sg.compute(ph, sg.Residency.Host)
    sg.compute(pd, sg.Residency.Device)
    sg.sync_to_host(pd)
    assert bits_equal(oh.values, od.values)


def test_device_residency_chain_matches_host_chain(sg, orc):
    """Config 1 pattern (10 x compute+swap) with Residency.Device: data stays
    in HBM between applications; one sync at the end."""
    rng = np.random.default_rng(7)
    inp = rng.uniform(-1, 1, (64, 64))
    dx = TWO_PI / 64
    cx = 1.0 / (dx * dx)
    w = [0.0, cx, 0.0, cx, -2 * cx - 2 * cx, cx, 0.0, cx, 0.0]
    a, b = sg.Grid2D.from_array(inp.copy()), sg.Grid2D(64, 64)
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, sg.WeightStencil(sg.Extents(1, 1, 1, 1), w),
                          a, b, 1, 1)
    for k in range(10):
        sg.compute(plan, sg.Residency.Device)
        if k < 9:
            sg.swap_plan(plan)
    sg.sync_to_host(plan)
    want = inp
    for _ in range(10):
        want = orc.stencil(want, (1, 1, 1, 1), w)
    assert bits_equal(plan.output().values, want)


def test_concurrent_plans_on_disjoint_buffers(sg, orc):
    """test_stencil.cpp:527-555 — two host threads, 50 computes each."""
    import threading
    rng = np.random.default_rng(171)
    w = rng.uniform(-2, 2, 16)
    ins = [rng.uniform(-1, 1, (18, 24)) for _ in range(2)]
    plans, outs = [], []
    for x in ins:
        go = sg.Grid2D(24, 18)
        outs.append(go)
        plans.append(sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                                    sg.WeightStencil(sg.Extents(2, 1, 1, 2), list(w)),
                                    sg.Grid2D.from_array(x), go, 3, 2))

    def run(p):
        for _ in range(50):
            sg.compute(p)

    ts = [threading.Thread(target=run, args=(p,)) for p in plans]
    [t.start() for t in ts]
    [t.join() for t in ts]
    for x, go in zip(ins, outs):
        assert bits_equal(go.values, orc.stencil(x, (2, 1, 1, 2), w))


# ------------------------------------------- general shapes / alignments


def _general_cases():
    """Asymmetric windows up to 9 x 9 (every left/right and top/bottom split
    of a few widths/heights) — k_tma_g's territory."""
    cases = [(3, 1, 0, 0), (0, 2, 0, 0), (2, 1, 1, 2), (0, 1, 0, 1), (1, 0, 2, 0), (4, 0, 0, 4),
             (0, 0, 3, 1), (0, 0, 0, 2), (3, 2, 1, 0), (1, 3, 4, 2), (8, 0, 0, 0), (0, 0, 0, 8),
             (5, 3, 2, 6), (0, 8, 8, 0), (6, 2, 1, 1), (2, 2, 4, 3)]
    return cases


@pytest.mark.parametrize("ext", _general_cases())
@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("nx", [320, 97, 2053])
def test_general_kernel_asymmetric_and_odd_bitwise(sg, orc, ext, periodic, nx):
    """k_tma_g: asymmetric windows (test_stencil.cpp:557-568 generalised) and
    odd row pitches (rows at every 16 B phase), periodic and not, one column
    block and several — bitwise vs the oracle, frame untouched."""
    rng = np.random.default_rng(hash((ext, nx, periodic)) & 0xFFFF)
    l, r, t, b = ext
    ny = 41
    if l + r >= nx or t + b >= ny:
        pytest.skip("window wider than the grid")
    inp = rng.uniform(-1, 1, (ny, nx))
    w = rng.uniform(-2, 2, (l + r + 1) * (t + b + 1))
    sentinel = np.full_like(inp, -12345.678)
    got = run_gpu(sg, inp, ext, w, direction=direction_of(ext), periodic=periodic, out=sentinel,
                  expect_kind=2)
    want = orc.stencil(inp, ext, w, periodic=periodic, out=sentinel)
    assert bits_equal(got, want)


def test_reference_asymmetric_case_3_1_0_0(sg, orc):
    """test_stencil.cpp:557-568: X stencil {3,1,0,0} on a periodic grid equals
    the single-point evaluation everywhere."""
    rng = np.random.default_rng(557)
    inp = rng.uniform(-1, 1, (16, 64))
    w = [0.5, -1.0, 2.0, 0.25, -0.75]
    got = run_gpu(sg, inp, (3, 1, 0, 0), w, direction=0, expect_kind=2)
    assert bits_equal(got, orc.stencil(inp, (3, 1, 0, 0), w))


@pytest.mark.parametrize("fn,ext,ncoe", FUNCS)
def test_general_kernel_functions_misaligned_pointers(sg, orc, fn, ext, ncoe):
    """Device grids whose base pointers are 8 B off 16 B alignment (a view one
    element into an allocation) run k_tma_g, bitwise."""
    import torch
    rng = np.random.default_rng(77)
    ny, nx = 33, 256
    inp = rng.uniform(-1.5, 1.5, (ny, nx))
    coe = rng.uniform(-2, 2, max(ncoe, 1))[:ncoe]
    bi = torch.zeros(ny * nx + 1, dtype=torch.float64, device="cuda")
    bo = torch.zeros(ny * nx + 3, dtype=torch.float64, device="cuda")
    ti = bi[1:].view(ny, nx)
    to = bo[3:].view(ny, nx)
    ti.copy_(torch.from_numpy(inp))
    kind = sg.FunctionStencil(sg.Extents(*ext), fn, list(coe))
    for periodic in (True, False):
        to.zero_()
        plan = sg.create_plan(direction_of(ext), sg.BoundaryMode.Periodic if periodic else sg.BoundaryMode.NonPeriodic,
                              kind, ti, to, 1, 1)
        assert plan.kernel_kind() == 2
        sg.compute(plan)
        want = orc.stencil(inp, ext, coe, periodic=periodic, fn=fn)
        assert bits_equal(to.cpu().numpy(), want)


@pytest.mark.parametrize("ext", [(1, 1, 1, 1), (3, 1, 0, 0), (2, 1, 1, 2), (4, 4, 4, 4)])
@pytest.mark.parametrize("nx", [255, 1026, 4099])
def test_general_kernel_fp32_odd_rows(sg, orc, ext, nx):
    """FP32 at every 16 B row phase (nx % 4 != 0): 1e-5 vs the FP64 oracle on
    the float-rounded input."""
    import torch
    rng = np.random.default_rng(nx)
    ny = 37
    inp32 = rng.uniform(-1, 1, (ny, nx)).astype(np.float32)
    l, r, t, b = ext
    w = rng.uniform(-2, 2, (l + r + 1) * (t + b + 1))
    ti = torch.from_numpy(inp32).cuda()
    to = torch.zeros_like(ti)
    plan = sg.create_plan(direction_of(ext), sg.BoundaryMode.Periodic, sg.WeightStencil(sg.Extents(*ext), list(w)),
                          ti, to, 1, 1)
    assert plan.kernel_kind() == (1 if (nx % 4 == 0 and l == r and t == b) else 2)
    sg.compute(plan)
    got = to.cpu().numpy().astype(np.float64)
    want = orc.stencil(inp32.astype(np.float64), ext, w)
    assert np.max(np.abs(got - want)) <= 1e-5 * np.max(np.abs(want))


def test_general_kernel_large_odd_grid_shift_property(sg, orc):
    """4097 x 3001 periodic {2,1,1,2}: bitwise vs the oracle, and the
    cyclic-shift equivariance (test_stencil.cpp:442-460) on the device."""
    import torch
    rng = np.random.default_rng(4097)
    w = rng.uniform(-1, 1, 16)
    inp = rng.uniform(-1, 1, (3001, 4097))
    ti = torch.from_numpy(inp).cuda()
    to, t2 = torch.empty_like(ti), torch.empty_like(ti)
    kind = sg.WeightStencil(sg.Extents(2, 1, 1, 2), list(w))
    p = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, kind, ti, to, 1, 1)
    assert p.kernel_kind() == 2
    sg.compute(p)
    assert bits_equal(to.cpu().numpy(), orc.stencil(inp, (2, 1, 1, 2), w))
    sh = torch.roll(ti, shifts=(17, -301), dims=(0, 1)).contiguous()
    p2 = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, kind, sh, t2, 1, 1)
    sg.compute(p2)
    assert torch.equal(torch.roll(to, shifts=(17, -301), dims=(0, 1)), t2)


# ----------------------------------------------------------------- FP32


@pytest.mark.parametrize("fn,ext,ncoe", [(None, (1, 1, 1, 1), 9), ("fn_weighted_3x3", (1, 1, 1, 1), 9),
                                         ("ch_nonlinear_window", (1, 1, 1, 1), 9),
                                         (None, (2, 2, 0, 0), 5), (None, (2, 2, 2, 2), 25)])
def test_fp32_within_1e5_of_fp64_oracle(sg, orc, fn, ext, ncoe):
    """FP32 extension: 1e-5 relative (normwise) vs the FP64 oracle evaluated
    on the float-rounded inputs."""
    import torch
    rng = np.random.default_rng(3)
    ny, nx = 96, 256
    inp32 = rng.uniform(-1, 1, (ny, nx)).astype(np.float32)
    w = rng.uniform(-2, 2, ncoe)
    ti = torch.from_numpy(inp32).cuda()
    to = torch.zeros_like(ti)
    kind = sg.WeightStencil(sg.Extents(*ext), list(w)) if fn is None else sg.FunctionStencil(sg.Extents(*ext), fn, list(w))
    plan = sg.create_plan(direction_of(ext), sg.BoundaryMode.Periodic, kind, ti, to, 1, 1)
    assert plan.kernel_kind() == 1
    sg.compute(plan)
    got = to.cpu().numpy().astype(np.float64)
    want = orc.stencil(inp32.astype(np.float64), ext, w, fn="weights" if fn is None else fn)
    assert np.max(np.abs(got - want)) <= 1e-5 * np.max(np.abs(want))


# ------------------------------------------------------ large-size property


def test_large_grid_checksum_and_shift_property(sg, orc):
    """At a size the oracle still finishes quickly (2048 x 1536, 3x3 fn
    stencil, device-resident) compare bitwise; the size-independent cyclic
    shift property is checked at 8192 x 4096 on the device alone."""
    import torch
    rng = np.random.default_rng(4)
    w = rng.uniform(-1, 1, 9)
    inp = rng.uniform(-1, 1, (1536, 2048))
    ti = torch.from_numpy(inp).cuda()
    to = torch.empty_like(ti)
    kind = sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", list(w))
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, kind, ti, to, 1, 1)
    sg.compute(plan)
    assert bits_equal(to.cpu().numpy(), orc.stencil(inp, (1, 1, 1, 1), w, fn="fn_weighted_3x3"))
    big = torch.rand(4096, 8192, dtype=torch.float64, device="cuda") * 2 - 1
    o1, o2 = torch.empty_like(big), torch.empty_like(big)
    sh = torch.roll(big, shifts=(123, -777), dims=(0, 1)).contiguous()
    p1 = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, kind, big, o1, 1, 1)
    p2 = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, kind, sh, o2, 1, 1)
    sg.compute(p1)
    sg.compute(p2)
    assert torch.equal(torch.roll(o1, shifts=(123, -777), dims=(0, 1)), o2)


def test_config4_full_size_sampled_rows_bitwise(sg, orc):
    """BASELINE config 4 at its full size (32768^2 FP64, 8 GiB per field):
    sampled rows — the wrap rows 0 and ny-1, and random interior rows — are
    bitwise equal to the oracle."""
    import torch
    n = 32768
    rng = np.random.default_rng(44)
    w = list(rng.uniform(-1, 1, 9))
    g = torch.Generator(device="cuda").manual_seed(44)
    a = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g).mul_(2).sub_(1)
    b = torch.empty_like(a)
    kind = sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", w)
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, kind, a, b, 1, 1)
    sg.compute(plan)
    rows = [0, 1, 511, 512, n // 2, n - 2, n - 1] + list(rng.integers(0, n, 5))
    idx = sorted({(j + d) % n for j in rows for d in (-1, 0, 1)})
    host = {j: a[j].cpu().numpy() for j in idx}
    for j in rows:
        band = np.stack([host[(j - 1) % n], host[j], host[(j + 1) % n]])
        want = orc.stencil(band, (1, 1, 1, 1), w, fn="fn_weighted_3x3")[1]
        assert bits_equal(b[j].cpu().numpy(), want), j
    sg.destroy_plan(plan)
    del a, b
    torch.cuda.empty_cache()


def test_beyond_int32_element_count_fp32(sg, orc):
    """More than 2^31 points in one grid (32768 x 65600 FP32, 8.6 GB per
    field): 64-bit indexing — rows past element 2^31 match the FP64 oracle
    on the float inputs within the FP32 bar (1e-5 relative)."""
    import torch
    nx, ny = 32768, 65600
    assert nx * ny > 2 ** 31
    rng = np.random.default_rng(45)
    w = list(rng.uniform(-1, 1, 9))
    g = torch.Generator(device="cuda").manual_seed(45)
    a = torch.rand((ny, nx), dtype=torch.float32, device="cuda", generator=g).mul_(2).sub_(1)
    b = torch.empty_like(a)
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                          sg.WeightStencil(sg.Extents(1, 1, 1, 1), w), a, b, 1, 1)
    sg.compute(plan)
    rows = [0, 65535, 65536, ny - 2, ny - 1]
    for j in rows:
        band = np.stack([a[(j + d) % ny].cpu().numpy().astype(np.float64) for d in (-1, 0, 1)])
        want = orc.stencil(band, (1, 1, 1, 1), w)[1]
        got = b[j].cpu().numpy().astype(np.float64)
        assert np.max(np.abs(got - want)) <= 1e-5 * np.max(np.abs(want)), j
    sg.destroy_plan(plan)
    del a, b
    torch.cuda.empty_cache()


# ------------------------------------------- BASELINE configs in full, GPU


def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def test_config1_full_matches_reference_golden(sg, orc):
    """BASELINE config 1 exactly: 512^2 XY periodic Laplacian, 10 x
    (compute, swap) through host Grid2D buffers with Device residency
    between applications — sha256 of the result equals the reference's
    (tests/golden/golden.json, generated from oracle/_ref)."""
    import json
    from pathlib import Path
    g = json.loads((Path(__file__).resolve().parent / "golden" / "golden.json").read_text())["config1"]
    inp = orc.ch_initial_condition(512, 512, seed=1, amp=1.0)
    assert _sha(inp) == g["input_sha256"]
    w = [float.fromhex(h) for h in g["weights_hex"]]
    gi, go = sg.Grid2D.from_array(inp), sg.Grid2D(512, 512)
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, sg.WeightStencil(sg.Extents(1, 1, 1, 1), w),
                          gi, go, 1, 1)
    for k in range(10):
        sg.compute(plan, sg.Residency.Device if k < 9 else sg.Residency.Host)
        if k < 9:
            sg.swap_plan(plan)
    # after 10 computes and 9 swaps the last output is plan.output()
    assert _sha(plan.output().values) == g["sha256"]


def test_config2_full_bitwise_vs_reference(sg, ref):
    """BASELINE config 2 exactly: 4096 x 4096 batched 1D non-periodic
    4th-derivative (X, {1,-4,6,-4,1}/dx^4), device vs the unmodified
    reference compute(), every point incl. the untouched frame."""
    import os
    import torch
    n = 4096
    dx = 2 * np.pi / n
    s4 = 1.0 / dx ** 4
    w = [s4, -4 * s4, 6 * s4, -4 * s4, s4]
    inp = np.random.default_rng(2).uniform(-1, 1, (n, n))
    frame = np.full((n, n), -12345.678)
    a = torch.from_numpy(inp).cuda()
    b = torch.from_numpy(frame).cuda()
    plan = sg.create_plan(sg.Direction.X, sg.BoundaryMode.NonPeriodic, sg.WeightStencil(sg.Extents(2, 2, 0, 0), w),
                          a, b, 1, 1)
    sg.compute(plan)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    want = ref.stencil(inp, (2, 2, 0, 0), w, direction=0, periodic=False, out=frame, tiles=cores, workers=cores)
    assert bits_equal(b.cpu().numpy(), want)


def test_config4_full_bitwise_vs_reference(sg, ref):
    """BASELINE config 4 (FP64) exactly: 32768^2 XY periodic 9-point user
    function (fn_weighted_3x3), every one of the 2^30 points bitwise equal to
    the unmodified reference compute() on this host's cores."""
    import os
    import torch
    n = 32768
    rng = np.random.default_rng(4)
    w = list(rng.uniform(-1, 1, 9))
    g = torch.Generator(device="cuda").manual_seed(4)
    a = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g).mul_(2).sub_(1)
    b = torch.empty_like(a)
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                          sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", w), a, b, 1, 1)
    sg.compute(plan)
    inp = a.cpu().numpy()
    got = b.cpu().numpy()
    del a, b
    torch.cuda.empty_cache()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    want = ref.stencil(inp, (1, 1, 1, 1), w, fn="fn_weighted_3x3", tiles=cores, workers=cores)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_config4_full_fp32_within_1e5_of_reference(sg, ref):
    """BASELINE config 4, FP32 half: 32768^2 XY periodic fn_weighted_3x3 in
    FP32 against the reference (FP64) on the float-rounded input, normwise
    max |err| <= 1e-5 max |ref| over all 2^30 points (north-star bar)."""
    import os
    import torch
    n = 32768
    w = list(np.random.default_rng(40).uniform(-1, 1, 9))
    g = torch.Generator(device="cuda").manual_seed(40)
    a = torch.rand((n, n), dtype=torch.float32, device="cuda", generator=g).mul_(2).sub_(1)
    b = torch.empty_like(a)
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                          sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", w), a, b, 1, 1)
    sg.compute(plan)
    inp = a.cpu().numpy().astype(np.float64)
    got = b.cpu().numpy()
    del a, b
    torch.cuda.empty_cache()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    want = ref.stencil(inp, (1, 1, 1, 1), w, fn="fn_weighted_3x3", tiles=cores, workers=cores)
    err = float(np.max(np.abs(got.astype(np.float64) - want)))
    assert err <= 1e-5 * float(np.max(np.abs(want)))


@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("ext,shape", [((1, 1, 1, 1), (64, 256)), ((3, 3, 3, 3), (64, 512)),
                                       ((4, 4, 4, 4), (72, 512)), ((3, 3, 0, 0), (40, 256)),
                                       ((0, 0, 2, 2), (48, 128)), ((1, 2, 0, 1), (33, 101))])
def test_fp32_paths_and_frames(sg, orc, periodic, ext, shape):
    """FP32 on every kernel path (TMA fast path incl. the tall-window
    accumulators, X-only, Y-only, and the generic kernel for asymmetric
    extents / odd sizes), periodic and not: within 1e-5 (normwise) of the
    FP64 oracle on the float inputs; non-periodic frames stay untouched."""
    import torch
    rng = np.random.default_rng(sum(ext) * 7 + periodic)
    ny, nx = shape
    inp32 = rng.uniform(-1, 1, (ny, nx)).astype(np.float32)
    W = (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
    w = rng.uniform(-2, 2, W)
    sentinel = np.float32(-12345.678)
    ti = torch.from_numpy(inp32).cuda()
    to = torch.full_like(ti, float(sentinel))
    mode = sg.BoundaryMode.Periodic if periodic else sg.BoundaryMode.NonPeriodic
    plan = sg.create_plan(direction_of(ext), mode, sg.WeightStencil(sg.Extents(*ext), list(w)), ti, to, 1, 1)
    sg.compute(plan)
    got = to.cpu().numpy()
    want = orc.stencil(inp32.astype(np.float64), ext, w, periodic=periodic,
                       out=np.full((ny, nx), float(sentinel)))
    if not periodic:
        frame = np.ones((ny, nx), bool)
        frame[ext[2]:ny - ext[3], ext[0]:nx - ext[1]] = False
        assert np.all(got[frame] == sentinel)
        inner = ~frame
    else:
        inner = np.ones((ny, nx), bool)
    err = np.max(np.abs(got[inner].astype(np.float64) - want[inner]))
    assert err <= 1e-5 * np.max(np.abs(want[inner]))


@pytest.mark.parametrize("ext", [(5, 5, 5, 5), (7, 2, 0, 9), (0, 12, 3, 3), (30, 29, 30, 28), (40, 40, 1, 1)])
@pytest.mark.parametrize("periodic", [True, False])
def test_generic_kernel_wide_windows_bitwise(sg, orc, ext, periodic):
    """k_generic: windows past 9 x 9 — tiled through shared memory, or (tile
    over 48 KB: the 60 x 59 and 81 x 3 windows) per point from global
    memory; periodic wrap on odd grid sizes, frame untouched."""
    rng = np.random.default_rng(sum(ext) + periodic)
    l, r, t, b = ext
    nx, ny = 101, 67
    if l + r >= nx or t + b >= ny:
        pytest.skip("window wider than the grid")
    inp = rng.uniform(-1, 1, (ny, nx))
    w = rng.uniform(-1, 1, (l + r + 1) * (t + b + 1))
    sentinel = np.full_like(inp, -12345.678)
    got = run_gpu(sg, inp, ext, w, direction=direction_of(ext), periodic=periodic, out=sentinel, expect_kind=0)
    want = orc.stencil(inp, ext, w, periodic=periodic, out=sentinel)
    assert bits_equal(got, want)
