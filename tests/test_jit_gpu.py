"""GPU parity of window functions registered from source (NVRTC-compiled into
the library's kernels). The reference's StencilFunction is arbitrary user
code (stencil.hpp:20-25); its loops call it per point with the window
(function_rows, stencil.cpp:96-126). FP64 results must equal a host
evaluation of the same expression bitwise: here numpy evaluates it
elementwise in the same operation order (IEEE, no contraction), and the
built-in twin of fn_weighted_3x3 must be matched exactly."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

WEIGHTED_3X3 = """
double acc = 0.0;  // tests/test_stencil.cpp:88-93
for (int q = 0; q < 3; ++q)
  for (int p = 0; p < 3; ++p) acc += coe[q * 3 + p] * window[q * rowStride + p];
return acc;
"""
# a function none of the built-in twins computes (reads its whole window)
NOVEL = """
const T c = window[rowStride + 1];
T acc = c * c * coe[0];
acc += (window[0] - window[2 * rowStride + 2]) * coe[1];
acc += window[rowStride] * window[rowStride + 2] - coe[2];
return acc;
"""


def novel_numpy(inp, coe, periodic=True):
    """NOVEL evaluated with numpy in the same order (3x3 window, extents 1)."""
    ny, nx = inp.shape
    out = np.zeros_like(inp)
    if periodic:
        def sh(dj, di):
            return np.roll(np.roll(inp, -dj, axis=0), -di, axis=1)
        c = sh(0, 0)
        acc = c * c * coe[0]
        acc = acc + (sh(-1, -1) - sh(1, 1)) * coe[1]
        acc = acc + (sh(0, -1) * sh(0, 1) - coe[2])
        return acc
    c = inp[1:-1, 1:-1]
    acc = c * c * coe[0]
    acc = acc + (inp[:-2, :-2] - inp[2:, 2:]) * coe[1]
    acc = acc + (inp[1:-1, :-2] * inp[1:-1, 2:] - coe[2])
    out[1:-1, 1:-1] = acc
    return out


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                                                 np.ascontiguousarray(b).view(np.uint64))


@pytest.fixture(scope="module")
def jit_ids(sg):
    return {"w3": sg.register_function_source("src_weighted_3x3", WEIGHTED_3X3),
            "novel": sg.register_function_source("src_novel", NOVEL)}


def run(sg, inp, ext, fn, coe, periodic=True, out=None):
    import torch
    ti = torch.from_numpy(inp).cuda()
    to = torch.from_numpy(np.zeros_like(inp) if out is None else out.copy()).cuda()
    e = sg.Extents(*ext)
    d = 0 if ext[2] == ext[3] == 0 else (1 if ext[0] == ext[1] == 0 else 2)
    plan = sg.create_plan(d, sg.BoundaryMode.Periodic if periodic else sg.BoundaryMode.NonPeriodic,
                          sg.FunctionStencil(e, fn, list(coe)), ti, to, 1, 1)
    kind = plan.kernel_kind()
    sg.compute(plan)
    return to.cpu().numpy(), kind


@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("nx,kind", [(320, 1), (97, 2), (2051, 2)])
def test_source_function_equals_builtin_twin(sg, jit_ids, periodic, nx, kind):
    """The reference's fn_weighted_3x3 from source == the compiled-in twin,
    bitwise, through k_tma (aligned rows) and k_tma_g (odd rows)."""
    rng = np.random.default_rng(nx)
    inp = rng.uniform(-1, 1, (45, nx))
    coe = rng.uniform(-2, 2, 9)
    got, k = run(sg, inp, (1, 1, 1, 1), "src_weighted_3x3", coe, periodic)
    want, _ = run(sg, inp, (1, 1, 1, 1), "fn_weighted_3x3", coe, periodic)
    assert k == kind
    assert bits_equal(got, want)


@pytest.mark.parametrize("periodic", [True, False])
def test_novel_source_function_bitwise_vs_host_expression(sg, jit_ids, periodic):
    rng = np.random.default_rng(7)
    inp = rng.uniform(-1.5, 1.5, (64, 256))
    coe = rng.uniform(-2, 2, 3)
    got, k = run(sg, inp, (1, 1, 1, 1), "src_novel", coe, periodic)
    assert k == 1
    assert bits_equal(got, novel_numpy(inp, coe, periodic))


def test_source_function_wide_window_generic_and_asymmetric(sg, jit_ids, orc):
    """The same function on windows it does not fill: an asymmetric one
    (k_tma_g) and one past 9 x 9 (k_generic). With rowStride = W the 3x3
    body reads the window's top-left 3 x 3 block, i.e. the weighted sum of
    the points (i - left + p, j - top + q) — the oracle's weight stencil on
    the same window with the other weights zero gives the same value."""
    rng = np.random.default_rng(11)
    inp = rng.uniform(-1, 1, (40, 130))
    coe = rng.uniform(-2, 2, 9)
    for ext, kind in (((2, 1, 1, 2), 2), ((5, 5, 5, 5), 0)):
        l, r, t, b = ext
        W, H = l + r + 1, t + b + 1
        got, k = run(sg, inp, ext, "src_weighted_3x3", coe)
        assert k == kind
        w = np.zeros(W * H)
        for q in range(3):
            w[q * W:q * W + 3] = coe[q * 3:q * 3 + 3]
        want = orc.stencil(inp, ext, w)
        # same terms, same order; the zero-weight taps add +0.0 exactly
        assert bits_equal(got, want)


def test_source_function_fp32(sg, jit_ids):
    import torch
    rng = np.random.default_rng(5)
    inp = rng.uniform(-1, 1, (50, 203)).astype(np.float32)
    coe = rng.uniform(-2, 2, 3)
    ti = torch.from_numpy(inp).cuda()
    to = torch.zeros_like(ti)
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                          sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "src_novel", list(coe)), ti, to, 1, 1)
    sg.compute(plan)
    want = novel_numpy(inp.astype(np.float64), coe.astype(np.float32).astype(np.float64))
    got = to.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(got - want) <= 1e-5 * np.linalg.norm(want)


def test_source_function_host_grids_and_workers(sg, jit_ids):
    """Host Grid2D plans (Residency::Host) and numWorkers > 1 (y-slabs on
    several GPUs, or several workers per GPU with the modulo device map) run
    the source function too, bitwise."""
    rng = np.random.default_rng(9)
    inp = rng.uniform(-1, 1, (60, 128))
    coe = rng.uniform(-2, 2, 3)
    want = novel_numpy(inp, coe)
    old = sg.get_device_map()
    sg.set_device_map("modulo")
    try:
        for workers in (1, 3):
            gi, go = sg.Grid2D.from_array(inp.copy()), sg.Grid2D.from_array(np.zeros_like(inp))
            plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                                  sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "src_novel", list(coe)), gi, go, 1,
                                  workers)
            sg.compute(plan)
            assert bits_equal(go.values, want)
    finally:
        sg.set_device_map(old)
