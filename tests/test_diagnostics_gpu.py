"""GPU: Cahn-Hilliard diagnostics on the device.
simpson_mean / s_metric bitwise vs the reference library; k1_metric within
1e-10 relative (cuFFT vs the reference's radix-2 FFT); the reference's KATs
(test_cahn_hilliard.cpp:320-366) and run()'s cadence (:475-505)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TWO_PI = 2 * math.pi


def grid(sg, f, n=64):
    dx = TWO_PI / n
    x = np.arange(n) * dx
    g = sg.Grid2D(n, n, dx, dx)
    g.values = np.ascontiguousarray(np.broadcast_to(f(x[None, :], x[:, None]), (n, n)), dtype=np.float64)
    return g


def test_simpson_and_s_metric_kats(sg):
    c = grid(sg, lambda x, y: 0.77 + 0 * x)
    assert sg.simpson_mean(c) == pytest.approx(0.77, rel=1e-13)
    s = grid(sg, lambda x, y: np.sin(x))
    assert abs(sg.simpson_mean(s)) <= 1e-14
    s2 = grid(sg, lambda x, y: np.sin(x) ** 2)
    assert sg.simpson_mean(s2) == pytest.approx(0.5, rel=1e-10)
    with pytest.raises(sg.InvalidArgument):
        sg.simpson_mean(sg.Grid2D(15, 16))
    assert sg.s_metric(sg.Grid2D(16, 16)) == 1.0
    one = sg.Grid2D(16, 16)
    one.values[:] = 1.0
    with pytest.raises(sg.DomainError):
        sg.s_metric(one)
    half = sg.Grid2D(16, 16)
    half.values[:] = 0.5
    assert sg.s_metric(half) == pytest.approx(4.0 / 3.0, rel=1e-13)


def test_k1_single_mode_kats(sg):
    cx = grid(sg, lambda x, y: np.cos(x))
    assert abs(sg.k1_metric(cx) - 1.0) <= 1e-12
    c4 = grid(sg, lambda x, y: np.cos(4.0 * y))
    assert abs(sg.k1_metric(c4) - 4.0) <= 1e-12
    cx.values *= 3.7
    assert abs(sg.k1_metric(cx) - 1.0) <= 1e-12
    with pytest.raises(sg.DomainError):
        sg.k1_metric(sg.Grid2D(64, 64, TWO_PI / 64, TWO_PI / 64))


def test_diagnostics_vs_reference(sg, ref):
    p = sg.CHParams(nx=128, ny=64)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    st = sg.CHStepper(p)
    st.step_many(30)
    d = st.diagnostics()
    s_ref, k_ref = ref.ch_diagnostics(st.field().values, p.dx(), p.dy())
    assert d.s == s_ref  # bitwise
    assert d.k1Inv == pytest.approx(k_ref, rel=1e-10)
    assert d.t == 30 * p.dt


def test_run_cadence(sg):
    p = sg.CHParams(nx=16, ny=16)
    p.dt = 0.1 * p.dx()
    p.T = p.dt
    p.icAmplitude = 0.0
    rows = []
    sg.run(p, 1, 1, sg.RunSink(diagEvery=1, onDiagnostics=rows.append))
    assert len(rows) == 2 and rows[0].t == 0.0 and rows[1].t == p.dt
    assert all(r.s == 1.0 for r in rows)
    p.T = 10.5 * p.dt
    snaps = []
    sg.run(p, 1, 1, sg.RunSink(diagEvery=0, snapEvery=5, onSnapshot=lambda g, s, t: snaps.append(s)))
    assert snaps == [0, 5, 10]


def _simpson_np(v, square=False):
    """composite Simpson mean in the reference's order (cahn_hilliard.cpp:
    161-176): per row a left-to-right sum (np.cumsum accumulates
    sequentially), then rows in order."""
    ny, nx = v.shape
    f = v * v if square else v
    wx = np.where(np.arange(nx) % 2 == 1, 4.0, 2.0)
    wy = np.where(np.arange(ny) % 2 == 1, 4.0, 2.0)
    row = np.cumsum(wx[None, :] * f, axis=1)[:, -1]
    return np.cumsum(wy * row)[-1] / (9.0 * float(nx) * float(ny))


@pytest.mark.parametrize("nx,ny", [(2, 2), (16, 16), (18, 6), (32, 64), (66, 34), (96, 40), (128, 16),
                                   (2048, 256), (256, 2048), (4096, 8)])
def test_simpson_bitwise_over_shapes(sg, nx, ny):
    """The device Simpson reduction (one warp per 32 rows, chunks fetched two
    ahead) keeps the reference's summation order on every shape: ragged
    chunks (nx not a multiple of 32), fewer rows than a warp, many chunks."""
    v = np.random.default_rng(nx * 7 + ny).uniform(-1, 1, (ny, nx))
    g = sg.Grid2D(nx, ny)
    g.values = v
    assert sg.simpson_mean(g) == _simpson_np(v)


@pytest.mark.parametrize("nx,ny", [(16, 16), (32, 64), (128, 16), (1024, 512)])
def test_s_metric_bitwise_vs_reference_shapes(sg, ref, nx, ny):
    v = np.random.default_rng(nx + ny).uniform(-1, 1, (ny, nx))
    g = sg.Grid2D(nx, ny, TWO_PI / nx, TWO_PI / ny)
    g.values = v
    s_ref, _ = ref.ch_diagnostics(v, TWO_PI / nx, TWO_PI / ny)
    assert sg.s_metric(g) == s_ref
