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


def _solve(sg, m, rhs):
    """Device solve of a copy of rhs (n, B) with a fresh factor of m."""
    import torch
    f = sg.PeriodicPentaFactor(m) if m.periodic else sg.PentaFactor(m)
    t = torch.from_numpy(np.ascontiguousarray(rhs, dtype=np.float64).copy()).cuda()
    f.solve_in_place(t)
    return t.cpu().numpy()


def _zero_corners(m):
    """penta.hpp:15-20: the cyclic wrap slots."""
    n = m.n
    m.secondSub[0, :] = m.secondSub[1, :] = m.sub[0, :] = 0.0
    m.secondSuper[n - 2, :] = m.super[n - 1, :] = m.secondSuper[n - 1, :] = 0.0


def test_zero_corner_periodic_equals_nonperiodic(sg):
    """test_penta.cpp:161-174: a periodic batch whose wrap couplings are zero
    solves to the same bits as the non-periodic batch."""
    m = random_batch(sg, 24, 40, True, 21)
    _zero_corners(m)
    rhs = np.random.default_rng(22).uniform(-1, 1, (40, 24))
    mn = sg.PentaBatch(24, 40, False)
    for a, b in zip(mn.bands(), m.bands()):
        a[:] = b
    assert bits_equal(_solve(sg, m, rhs), _solve(sg, mn, rhs))


@pytest.mark.parametrize("periodic", [False, True])
def test_system_permutation_bitwise(sg, periodic):
    """test_penta.cpp:225-247: permuting the systems of a batch permutes the
    solutions, bit for bit (systems are independent)."""
    B, n = 37, 29
    m = random_batch(sg, B, n, periodic, 31)
    rhs = np.random.default_rng(32).uniform(-1, 1, (n, B))
    perm = np.random.default_rng(33).permutation(B)
    mp = sg.PentaBatch(B, n, periodic)
    for a, b in zip(mp.bands(), m.bands()):
        a[:] = b[:, perm]
    assert bits_equal(_solve(sg, mp, rhs[:, perm]), _solve(sg, m, rhs)[:, perm])


@pytest.mark.parametrize("periodic", [False, True])
def test_batch_equals_single_system_solves(sg, periodic):
    """test_penta.cpp:306-316 (parallel == serial): the batched device solve
    equals solving every system as a batch of one, bitwise."""
    B, n = 9, 33
    m = random_batch(sg, B, n, periodic, 41)
    rhs = np.random.default_rng(42).uniform(-1, 1, (n, B))
    got = _solve(sg, m, rhs)
    for b in range(B):
        m1 = sg.PentaBatch(1, n, periodic)
        for a, band in zip(m1.bands(), m.bands()):
            a[:, 0] = band[:, b]
        assert bits_equal(_solve(sg, m1, rhs[:, b:b + 1])[:, 0], got[:, b])


def test_amortized_factor_equals_fresh(sg):
    """test_penta.cpp:294-304: one factor reused for several right-hand
    sides gives the same bits as a fresh factor per solve."""
    import torch
    m = random_batch(sg, 16, 48, True, 51)
    f = sg.PeriodicPentaFactor(m)
    rng = np.random.default_rng(52)
    for _ in range(4):
        rhs = rng.uniform(-1, 1, (48, 16))
        t = torch.from_numpy(rhs.copy()).cuda()
        f.solve_in_place(t)
        assert bits_equal(t.cpu().numpy(), _solve(sg, m, rhs))


def test_linearity(sg):
    """test_penta.cpp:249-263: solve(a x + b y) = a solve(x) + b solve(y)
    within 1e-12 (relative, normwise)."""
    m = random_batch(sg, 12, 50, True, 61)
    rng = np.random.default_rng(62)
    x, y = rng.uniform(-1, 1, (50, 12)), rng.uniform(-1, 1, (50, 12))
    a, b = 0.75, -1.25
    lhs = _solve(sg, m, a * x + b * y)
    rhs = a * _solve(sg, m, x) + b * _solve(sg, m, y)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(rhs))


def test_hyperdiffusion_preserves_the_mean(sg):
    """test_penta.cpp:278-292: rows of the periodic hyperdiffusion operator
    sum to 1 and it is circulant, so the solution keeps the mean of the
    right-hand side (1e-13)."""
    n, B = 64, 8
    m = sg.build_hyperdiffusion_operator(3.5, n, B, True)
    rhs = np.random.default_rng(71).uniform(-1, 1, (n, B))
    got = _solve(sg, m, rhs)
    assert np.max(np.abs(got.mean(axis=0) - rhs.mean(axis=0))) <= 1e-13
