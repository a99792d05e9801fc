"""GPU parity tests for the batched pentadiagonal solver (tests/test_penta.cpp
restated). Checker: the C restatement (bitwise-pinned to the reference) and
dense numpy solves for the residual KATs."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                                                 np.ascontiguousarray(b).view(np.uint64))


def random_batch(sg, B, n, periodic, seed, dominance=6.0):
    rng = np.random.default_rng(seed)
    m = sg.PentaBatch(B, n, periodic)
    for band in m.bands():
        band[:] = rng.uniform(-1, 1, (n, B))
    m.diag += dominance
    return m


def dense(m, b):
    n = m.n
    A = np.zeros((n, n))
    for r in range(n):
        for off, band in zip((-2, -1, 0, 1, 2), m.bands()):
            c = r + off
            if m.periodic:
                A[r, c % n] += band[r, b]
            elif 0 <= c < n:
                A[r, c] += band[r, b]
    return A


@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("B,n", [(1, 5), (7, 12), (33, 64), (300, 37)])
def test_random_batches_bitwise_vs_oracle(sg, orc, periodic, B, n):
    m = random_batch(sg, B, n, periodic, seed=B * 131 + n)
    rhs = sg.RhsBatch(B, n, np.random.default_rng(n).uniform(-1, 1, (n, B)))
    got = (sg.solve_periodic_batch if periodic else sg.solve_batch)(m, rhs).values
    want = orc.penta_solve(periodic, m.bands(), rhs.values)
    assert bits_equal(got, want)


def test_uniform_operator_path_bitwise(sg, orc):
    """All systems identical (the CH operator): device keeps n-vector factors."""
    for periodic in (False, True):
        m = sg.build_hyperdiffusion_operator(2.9e3, 256, 100, periodic)
        rhs = np.random.default_rng(3).uniform(-1, 1, (256, 100))
        got = (sg.solve_periodic_batch if periodic else sg.solve_batch)(m, sg.RhsBatch(100, 256, rhs)).values
        assert bits_equal(got, orc.penta_solve(periodic, m.bands(), rhs))


def test_dense_oracle_residuals(sg):
    """test_penta.cpp:105-114, 176-186, 265-276 — residual <= 1e-10."""
    for periodic in (False, True):
        for seed in range(20):
            B, n = 3, 9 + seed
            m = random_batch(sg, B, n, periodic, seed)
            rhs = np.random.default_rng(seed + 1).uniform(-1, 1, (n, B))
            x = (sg.solve_periodic_batch if periodic else sg.solve_batch)(m, sg.RhsBatch(B, n, rhs)).values
            for b in range(B):
                A = dense(m, b)
                assert np.max(np.abs(A @ x[:, b] - rhs[:, b])) <= 1e-10


def test_identity_and_sigma_zero(sg):
    """test_penta.cpp:96-103, 116-124 — identity / sigma = 0 operator is exact."""
    rhs = np.random.default_rng(1).uniform(-1, 1, (16, 5))
    for periodic in (False, True):
        m = sg.build_hyperdiffusion_operator(0.0, 16, 5, periodic)
        got = (sg.solve_periodic_batch if periodic else sg.solve_batch)(m, sg.RhsBatch(5, 16, rhs)).values
        assert bits_equal(got, rhs)


def test_circulant_eigenvector(sg):
    """test_penta.cpp:188-199 — cos(k r) / lambda, lambda = 1 + s(6 - 8cos k + 2cos 2k)."""
    n, s = 64, 0.37
    m = sg.build_hyperdiffusion_operator(s, n, 2, True)
    for kk in (1, 3, 7):
        k = 2 * math.pi * kk / n
        v = np.cos(k * np.arange(n))
        lam = 1 + s * (6 - 8 * math.cos(k) + 2 * math.cos(2 * k))
        x = sg.solve_periodic_batch(m, sg.RhsBatch(2, n, np.stack([v, v], axis=1))).values
        assert np.max(np.abs(x[:, 0] - v / lam)) <= 1e-13


def test_zero_pivot_reports_system(sg):
    """test_penta.cpp:201-212 — zero pivot in system 1 -> PentaSolveError(1)."""
    m = sg.PentaBatch(3, 6, False)
    m.diag[:] = 1.0
    m.diag[0, 1] = 0.0
    with pytest.raises(sg.PentaSolveError) as ei:
        sg.solve_batch(m, sg.RhsBatch(3, 6))
    assert ei.value.system == 1


def test_shape_errors(sg):
    m = sg.build_hyperdiffusion_operator(0.1, 8, 2, False)
    with pytest.raises(sg.InvalidArgument):
        sg.solve_periodic_batch(m, sg.RhsBatch(2, 8))
    with pytest.raises(sg.InvalidArgument):
        sg.solve_batch(m, sg.RhsBatch(3, 8))
    with pytest.raises(sg.InvalidArgument):
        sg.PentaBatch(1, 4, False)


def test_operator_rows_kat(sg):
    """test_penta.cpp:126-159 — sigma = 0.25 rows; row sums 1."""
    m = sg.build_hyperdiffusion_operator(0.25, 8, 1, True)
    assert m.diag[3, 0] == 2.5 and m.sub[3, 0] == -1.0 and m.secondSub[3, 0] == 0.25
    total = sum(b[:, 0] for b in m.bands())
    assert np.all(total == 1.0)


def test_device_resident_rhs(sg, orc):
    import torch
    m = random_batch(sg, 64, 40, True, 5)
    rhs = np.random.default_rng(2).uniform(-1, 1, (40, 64))
    f = sg.PeriodicPentaFactor(m)
    t = torch.from_numpy(rhs.copy()).cuda()
    f.solve_in_place(t)
    assert bits_equal(t.cpu().numpy(), orc.penta_solve(True, m.bands(), rhs))


@pytest.mark.parametrize("periodic", [False, True])
def test_uniform_large_batch_bitwise(sg, orc, periodic):
    """A uniform operator over more systems than one CTA per SM (B = 8192:
    the resident-turn sweep's 64-row-stage geometry, two CTAs per SM),
    device-resident rhs, bitwise vs the oracle."""
    import torch
    B, n = 8192, 96
    m = sg.build_hyperdiffusion_operator(2.5, n, B, periodic)
    rhs = np.random.default_rng(8).uniform(-1, 1, (n, B))
    f = sg.PeriodicPentaFactor(m) if periodic else sg.PentaFactor(m)
    t = torch.from_numpy(rhs.copy()).cuda()
    f.solve_in_place(t)
    assert bits_equal(t.cpu().numpy(), orc.penta_solve(periodic, m.bands(), rhs))
