"""Streamed (out-of-core) host plans: no device mirrors, the grid streams
through a ring of row-chunk buffers (sg.h). Forced at small sizes with
SG_STREAM_PLANS=1 and tiny chunks (SG_STREAM_ROWS), so chunks are shorter
than the window, wrap around periodic grids and end mid-grid; results must
be bitwise the oracle's (FP64), the non-periodic output frame untouched."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture
def streamed(monkeypatch):
    def set_rows(rows):
        monkeypatch.setenv("SG_STREAM_PLANS", "1")
        monkeypatch.setenv("SG_STREAM_ROWS", str(rows))
    return set_rows


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def direction_of(ext):
    l, r, t, b = ext
    return 0 if t == b == 0 else (1 if l == r == 0 else 2)


CASES = [((1, 1, 1, 1), None, 9), ((2, 2, 0, 0), None, 5), ((0, 0, 2, 2), None, 5), ((4, 4, 4, 4), None, 81),
         ((3, 1, 0, 0), None, 5), ((2, 1, 1, 2), None, 16), ((0, 0, 3, 1), None, 5),
         ((1, 1, 1, 1), "fn_weighted_3x3", 9), ((1, 1, 1, 1), "ch_nonlinear_window", 9)]


@pytest.mark.parametrize("rows", [1, 3, 7, 64])
@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("ext,fn,nv", CASES)
def test_streamed_plan_bitwise(sg, orc, streamed, rows, periodic, ext, fn, nv):
    streamed(rows)
    rng = np.random.default_rng(rows * 31 + nv)
    ny, nx = 45, 130
    inp = rng.uniform(-1, 1, (ny, nx))
    vals = rng.uniform(-2, 2, nv)
    sentinel = np.full_like(inp, -12345.678)
    gi, go = sg.Grid2D.from_array(inp.copy()), sg.Grid2D.from_array(sentinel.copy())
    e = sg.Extents(*ext)
    kind = sg.WeightStencil(e, list(vals)) if fn is None else sg.FunctionStencil(e, fn, list(vals))
    plan = sg.create_plan(direction_of(ext), sg.BoundaryMode.Periodic if periodic else sg.BoundaryMode.NonPeriodic,
                          kind, gi, go, 1, 1)
    sg.compute(plan)
    want = orc.stencil(inp, ext, vals, periodic=periodic, fn="weights" if fn is None else fn, out=sentinel)
    assert bits_equal(go.values, want)
    # swap + a second application (compute / swap / compute, test_stencil.cpp:227-249)
    sg.swap_plan(plan)
    sg.compute(plan, sg.Residency.Device)  # behaves as Host on a streamed plan
    want2 = orc.stencil(want, ext, vals, periodic=periodic, fn="weights" if fn is None else fn, out=inp)
    assert bits_equal(gi.values, want2)
    sg.destroy_plan(plan)


def test_streamed_plan_fp32_and_odd_width(sg, orc, streamed):
    import torch  # noqa: F401  (CUDA context)
    streamed(5)
    rng = np.random.default_rng(3)
    inp = rng.uniform(-1, 1, (33, 97)).astype(np.float32)
    w = rng.uniform(-2, 2, 9)
    gi = sg.Grid2D.from_array(inp.copy())
    go = sg.Grid2D.from_array(np.zeros_like(inp))
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, sg.WeightStencil(sg.Extents(1, 1, 1, 1), list(w)),
                          gi, go, 1, 1)
    sg.compute(plan)
    want = orc.stencil(inp.astype(np.float64), (1, 1, 1, 1), w)
    assert np.max(np.abs(go.values.astype(np.float64) - want)) <= 1e-5 * np.max(np.abs(want))


def test_large_nonperiodic_host_compute_pipelined(sg, orc):
    """A mirrored plan's large non-periodic Residency::Host compute (>= 64
    MiB: BASELINE config 2's 4096^2 batched 1D 4th derivative through host
    Grid2D fields) takes the streamed pipeline: bitwise, frame untouched,
    and a following Device-residency compute still sees the right input."""
    n = 4096
    dx = 2 * np.pi / n
    s4 = 1.0 / dx ** 4
    w = [s4, -4 * s4, 6 * s4, -4 * s4, s4]
    inp = np.random.default_rng(2).uniform(-1, 1, (n, n))
    frame = np.full((n, n), -12345.678)
    gi, go = sg.Grid2D.from_array(inp.copy()), sg.Grid2D.from_array(frame.copy())
    plan = sg.create_plan(sg.Direction.X, sg.BoundaryMode.NonPeriodic, sg.WeightStencil(sg.Extents(2, 2, 0, 0), w),
                          gi, go, 1, 1)
    sg.compute(plan)
    want = orc.stencil(inp, (2, 2, 0, 0), w, periodic=False, out=frame)
    assert bits_equal(go.values, want)
    sg.compute(plan, sg.Residency.Device)  # mirrors were stale: re-uploaded
    sg.sync_to_host(plan)
    assert bits_equal(go.values, want)
