"""CPU: pin the oracle before trusting it.

1. The C restatement (oracle/liboracle.so) reproduces every committed golden
   fixture (generated from the unmodified reference by
   tests/golden/make_golden.py) BITWISE.
2. Where the reference library is available (oracle/_ref), the restatement
   matches it bitwise on fresh random cases (stencil, penta, CH).
3. The reference's own known-answer tests (test_grid.cpp, test_stencil.cpp,
   test_penta.cpp, test_cahn_hilliard.cpp) hold for the restatement.
"""
import hashlib
import json
import math
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"
TWO_PI = 2.0 * math.pi
INV_FN = {0: "weights", 1: "ch_nonlinear_window", 2: "central_difference_window", 3: "fn_center",
          4: "fn_central_second", 5: "fn_lap_cube_diff_first", 6: "fn_weighted_3x3"}


def bits_equal(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def golden():
    return json.loads((GOLD / "golden.json").read_text())


# ------------------------------------------------------------- 1. golden


def test_stencil_golden_cases(orc):
    z = np.load(GOLD / "stencil_cases.npz")
    for k in range(int(z["count"][0])):
        d, per, fid, *e = (int(v) for v in z[f"c{k}_meta"])
        inp = z[f"c{k}_in"]
        got = orc.stencil(inp, e, z[f"c{k}_w"], periodic=bool(per), fn=INV_FN[fid],
                          out=np.full_like(inp, -12345.678))
        assert bits_equal(got, z[f"c{k}_out"]), k


def test_config1_golden(orc, golden):
    g = golden["config1"]
    inp = orc.ch_initial_condition(512, 512, seed=1, amp=1.0)
    assert sha(inp) == g["input_sha256"]
    w = [float.fromhex(h) for h in g["weights_hex"]]
    x = inp
    for _ in range(10):
        x = orc.stencil(x, (1, 1, 1, 1), w)
    assert sha(x) == g["sha256"]


def test_config2_small_golden(orc):
    z = np.load(GOLD / "config2_small.npz")
    got = orc.stencil(z["inp"], (2, 2, 0, 0), z["w"], periodic=False,
                      out=np.full_like(z["inp"], -12345.678))
    assert bits_equal(got, z["out"])


def test_penta_golden(orc):
    z = np.load(GOLD / "penta_cases.npz")
    for k in range(int(z["count"][0])):
        per, B, n = (int(v) for v in z[f"p{k}_meta"])
        bands = [z[f"p{k}_{c}"] for c in "ecdab"]
        assert bits_equal(orc.penta_solve(per, bands, z[f"p{k}_rhs"]), z[f"p{k}_x"]), k


def test_ch_golden(orc, golden):
    z = np.load(GOLD / "ch_32x16_10steps.npz")
    D, gamma, lx, ly, dt = z["params"]
    c0 = orc.ch_initial_condition(32, 16, seed=5)
    c, p = orc.ch_run(dict(D=D, gamma=gamma, lx=lx, ly=ly, dt=dt, nx=32, ny=16), 10, c0, c0)
    assert bits_equal(c, z["curr"]) and bits_equal(p, z["prev"])
    for key, g in golden["ch"].items():
        n = g["nx"]
        dt = float.fromhex(g["dt_hex"])
        c0 = orc.ch_initial_condition(n, n, seed=g["seed"])
        c, p = orc.ch_run(dict(D=1.0, gamma=0.01, lx=TWO_PI, ly=TWO_PI, dt=dt, nx=n, ny=n,
                               nonlinear=g["nonlinear"]), g["steps"], c0, c0)
        assert sha(c) == g["curr_sha256"], key
        assert sha(p) == g["prev_sha256"], key


def test_kats_golden(orc, golden):
    k = golden["kats"]
    for n in (64, 1024, 8192):
        dx = TWO_PI / n
        bw, nl = orc.ch_weights(dx, dx)
        assert [float(x).hex() for x in bw] == k[f"biharmonic_weights_{n}"]
        assert [float(x).hex() for x in nl] == k[f"nonlinear_coefficients_{n}"]
        assert sum(bw[:22]) + bw[22] == 0.0 or True  # row-major prefix sum is exactly 0 below
        acc = 0.0
        for x in bw:
            acc += x
        assert acc == 0.0  # test_cahn_hilliard.cpp:149-158
    for i, n, want in k["wrap"]:
        assert orc.wrap(i, n) == want
    for key, tiles in k["make_tiles"].items():
        ny, t = (int(v) for v in key.split("_"))
        assert [list(x) for x in orc.make_tiles(ny, t)] == tiles


# ------------------------------------------------- 2. live reference parity


def test_restatement_vs_reference_random_stencils(orc, ref):
    rng = np.random.default_rng(12345)
    for _ in range(150):
        nx, ny = (int(v) for v in rng.integers(1, 20, 2))
        d = int(rng.integers(0, 3))
        e = [0, 0, 0, 0]
        if d != 1:
            e[0], e[1] = (int(v) for v in rng.integers(0, min(4, nx - 1) + 1, 2))
        if d != 0:
            e[2], e[3] = (int(v) for v in rng.integers(0, min(4, ny - 1) + 1, 2))
        w = rng.uniform(-2, 2, (e[0] + e[1] + 1) * (e[2] + e[3] + 1))
        inp = rng.uniform(-2, 2, (ny, nx))
        for per in (True, False):
            o0 = rng.uniform(-1, 1, (ny, nx))
            a = orc.stencil(inp, e, w, periodic=per, out=o0)
            b = ref.stencil(inp, e, w, direction=d, periodic=per, out=o0, tiles=min(3, ny), workers=2)
            assert bits_equal(a, b)


def test_restatement_vs_reference_penta_and_ch(orc, ref):
    rng = np.random.default_rng(9)
    for per in (0, 1):
        for B, n in [(5, 11), (40, 64)]:
            bands = [rng.uniform(-1, 1, (n, B)) for _ in range(5)]
            bands[2] += 6.0
            rhs = rng.uniform(-1, 1, (n, B))
            assert bits_equal(orc.penta_solve(per, bands, rhs), ref.penta_solve(per, bands, rhs, workers=3))
    from oracle.oracle import ch_params
    for nx, ny, steps in [(16, 16, 4), (64, 32, 6)]:
        p = ch_params(nx, ny, seed=11)
        c_ref, p_ref = ref.ch_run(p, steps, tiles=2, workers=2)
        c0 = orc.ch_initial_condition(nx, ny, seed=11)
        c, pr = orc.ch_run(p, steps, c0, c0)
        assert bits_equal(c, c_ref) and bits_equal(pr, p_ref)


def test_ch_factor_tables_match_reference_operator(orc, ref):
    """The uniform factor (one system) equals the batched reference factor's
    behaviour: solving with B systems of the CH operator equals per-system
    uniform solves (SURVEY.md §8(a) key fact (i))."""
    n, B = 64, 9
    dx = TWO_PI / n
    dt = 0.1 * dx
    sigma = (2.0 / 3.0) * 1.0 * 0.01 * dt / ((dx * dx) * (dx * dx))
    bands = ref.hyperdiffusion_operator(sigma, n, B, True)
    rhs = np.random.default_rng(1).uniform(-1, 1, (n, B))
    assert bits_equal(orc.penta_solve(1, bands, rhs), ref.penta_solve(1, bands, rhs))
    t = orc.uniform_factor_tables(sigma, n)
    assert t["bad"] < 0 and np.all(np.isfinite(t["dInv"]))


# --------------------------------------------------- 3. reference KATs


def test_brute_force_kats(orc):
    """test_stencil.cpp:291-303 (cross derivative of i^2 j^2 == 4) and
    :278-289 identity."""
    i = np.arange(8, dtype=np.float64)
    g = (i[None, :] ** 2) * (i[:, None] ** 2)
    out = orc.stencil(g, (1, 1, 1, 1), [1, -2, 1, -2, 4, -2, 1, -2, 1], periodic=False)
    assert np.all(out[1:7, 1:7] == 4.0)
    x = np.random.default_rng(0).uniform(-1, 1, (11, 9))
    assert bits_equal(orc.stencil(x, (0, 0, 0, 0), [1.0]), x)


def test_penta_identity_and_circulant(orc):
    n, s = 32, 0.37
    bands = orc.hyperdiffusion_operator(s, n, 1, True)
    k = 2 * math.pi * 3 / n
    v = np.cos(k * np.arange(n))[:, None]
    lam = 1 + s * (6 - 8 * math.cos(k) + 2 * math.cos(2 * k))
    assert np.max(np.abs(orc.penta_solve(1, bands, v) - v / lam)) <= 1e-13
    eye = orc.hyperdiffusion_operator(0.0, 12, 3, False)
    r = np.random.default_rng(2).uniform(-1, 1, (12, 3))
    assert bits_equal(orc.penta_solve(0, eye, r), r)


def test_initial_condition_statistics(orc):
    """test_cahn_hilliard.cpp:76-100."""
    f = orc.ch_initial_condition(512, 512, seed=1, amp=0.1)
    assert np.max(np.abs(f)) <= 0.1
    assert abs(f.mean()) <= 3.0 * (0.1 / math.sqrt(3.0)) / 512.0
    assert np.all(orc.ch_initial_condition(8, 8, amp=0.0) == 0.0)
