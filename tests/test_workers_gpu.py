"""GPU: numWorkers -> GPUs behind the drop-in create_plan (stencil.hpp:90-92;
SPEC.md:12 maps cuSten's deviceNum onto the workers). A plan over host grids
with numWorkers = G splits the rows into make_tiles(ny, G) y-slabs, one per
worker/GPU. The box has one GPU, so the tests select the "modulo" device map
(G workers on GPU w % 1): the multi-worker machinery — per-worker slabs,
host-side halo rows, peer halo refreshes for device-resident inputs, the
row-chunk pipeline — runs exactly as on 8 GPUs, and every result must be
bitwise the oracle's (the reference's tile/worker invariance,
test_stencil.cpp:390-409)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SENTINEL = -12345.678


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                                                 np.ascontiguousarray(b).view(np.uint64))


@pytest.fixture
def modulo(sg):
    sg.set_device_map("modulo")
    yield
    sg.set_device_map("clip")


CASES = [  # (direction, periodic, extents, fn)
    ("XY", True, (1, 1, 1, 1), "fn_weighted_3x3"),
    ("XY", False, (2, 2, 2, 2), "weights"),
    ("X", False, (2, 2, 0, 0), "weights"),
    ("Y", True, (0, 0, 3, 1), "weights"),
    ("XY", True, (3, 1, 0, 2), "weights"),
]


def _kind(sg, ext, fn, rng):
    W = (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
    if fn == "weights":
        w = list(rng.uniform(-2, 2, W))
        return sg.WeightStencil(sg.Extents(*ext), w), w
    w = list(rng.uniform(-2, 2, 9))
    return sg.FunctionStencil(sg.Extents(*ext), fn, w), w


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("case", CASES)
def test_workers_bitwise_host_and_device_residency(sg, orc, modulo, G, case):
    d, periodic, ext, fn = case
    rng = np.random.default_rng(21 + G)
    nx, ny = 96, 40
    kind, w = _kind(sg, ext, fn, rng)
    x = rng.uniform(-1, 1, (ny, nx))
    gi, go = sg.Grid2D.from_array(x), sg.Grid2D(nx, ny)
    go.values[:] = SENTINEL
    mode = sg.BoundaryMode.Periodic if periodic else sg.BoundaryMode.NonPeriodic
    plan = sg.create_plan(getattr(sg.Direction, d), mode, kind, gi, go, 1, G)
    ws = plan.workers()
    assert len(ws) == G
    assert [(b, e) for _, b, e in ws] == sg.make_tiles(ny, G)
    # one synchronous application (Residency::Host)
    sg.compute(plan)
    want = orc.stencil(x, ext, w, periodic=periodic, fn=fn, out=np.full_like(x, SENTINEL))
    assert bits_equal(go.values, want)
    # three device-resident applications (halos refreshed between workers)
    cur = want
    ref_in, ref_out = want.copy(), x.copy()
    for k in range(3):
        sg.swap_plan(plan)
        sg.compute(plan, sg.Residency.Device)
        ref_out = orc.stencil(ref_in, ext, w, periodic=periodic, fn=fn, out=ref_out)
        ref_in, ref_out = ref_out, ref_in
    sg.sync_to_host(plan)
    cur = plan.output().values
    assert bits_equal(cur, ref_in)
    sg.destroy_plan(plan)


def test_workers_thinner_than_halo(sg, orc, modulo):
    """8 workers on 10 rows with a 7-row window: slabs of 1-2 rows whose halo
    rows come from several other workers (host rows, then peer refreshes)."""
    rng = np.random.default_rng(5)
    nx, ny, ext = 64, 10, (0, 0, 3, 3)
    w = list(rng.uniform(-1, 1, 7))
    x = rng.uniform(-1, 1, (ny, nx))
    gi, go = sg.Grid2D.from_array(x), sg.Grid2D(nx, ny)
    plan = sg.create_plan(sg.Direction.Y, sg.BoundaryMode.Periodic, sg.WeightStencil(sg.Extents(*ext), w),
                          gi, go, 1, 8)
    ref = x.copy()
    for _ in range(4):
        sg.compute(plan, sg.Residency.Device)
        sg.swap_plan(plan)
        ref = orc.stencil(ref, ext, w)
    sg.sync_to_host(plan)
    assert bits_equal(plan.input().values, ref)


@pytest.mark.parametrize("G", [2, 5])
def test_workers_pipelined_large_grid_equals_one_gpu(sg, modulo, G):
    """A 4096^2 grid (128 MB: the row-chunk H2D/compute/D2H pipeline per
    worker) — bitwise equal to the one-GPU plan, FP64 and FP32."""
    rng = np.random.default_rng(9)
    for dt in (np.float64, np.float32):
        x = rng.uniform(-1, 1, (4096, 4096)).astype(dt)
        w = list(rng.uniform(-1, 1, 9))
        kind = sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", w)
        outs = []
        for workers in (1, G):
            gi, go = sg.Grid2D.from_array(x), sg.Grid2D.from_array(np.zeros_like(x))
            plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, kind, gi, go, 1, workers)
            sg.compute(plan)
            outs.append(go.values.copy())
            sg.destroy_plan(plan)
        assert bits_equal(outs[0], outs[1])


def test_clip_map_uses_at_most_the_visible_gpus(sg):
    import torch
    sg.set_device_map("clip")
    x = np.zeros((16, 16))
    gi, go = sg.Grid2D.from_array(x), sg.Grid2D(16, 16)
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                          sg.WeightStencil(sg.Extents(1, 1, 1, 1), [0.0] * 4 + [1.0] + [0.0] * 4), gi, go, 1, 8)
    assert len(plan.workers()) == min(8, torch.cuda.device_count())
    with pytest.raises(sg.InvalidArgument):
        sg.set_device_map("round-robin")
