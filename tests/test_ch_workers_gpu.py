"""GPU: CHStepper(params, numTiles, numWorkers) with numWorkers -> GPUs
(cahn_hilliard.hpp:104-137). With G > 1 workers the stepper runs
config 5's distributed step from one process over G devices — the "modulo"
device map puts G workers on this box's one GPU, so the multi-GPU machinery
(per-worker slabs and streams, peer stores of the all-to-all blocks and halo
rows, cross-device event barriers, or the copy-engine form when the sweep
stage does not divide a slab) runs exactly as on 8 GPUs. Every field must be
bitwise the one-GPU stepper's (the reference's tile/worker invariance,
test_cahn_hilliard.cpp:453-465, acceptance.cpp:154-178)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                                                 np.ascontiguousarray(b).view(np.uint64))


@pytest.fixture
def modulo(sg):
    sg.set_device_map("modulo")
    yield
    sg.set_device_map("clip")


def params(sg, n, **kw):
    p = sg.CHParams(nx=n, ny=n)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    for k, v in kw.items():
        setattr(p, k, v)
    return p


@pytest.mark.parametrize("n,G,p2p", [(256, 2, True), (256, 8, False), (1024, 4, True), (1024, 8, True),
                                     (128, 3, False)])
def test_ch_workers_bitwise(sg, modulo, n, G, p2p):
    p = params(sg, n, seed=3)
    multi = sg.CHStepper(p, 1, G)
    g_eff, is_p2p = multi.workers()
    assert g_eff == (2 if G == 3 else G)  # the largest power of two <= G
    assert is_p2p == p2p
    single = sg.CHStepper(p)
    for steps in (1, 6):
        multi.step_many(steps)
        single.step_many(steps)
        assert bits_equal(multi.field().values, single.field().values)
        assert bits_equal(multi.previous_field().values, single.previous_field().values)
    assert multi.step_index() == 7 and multi.time() == single.time()
    dm, ds = multi.diagnostics(), single.diagnostics()
    assert (dm.t, dm.s) == (ds.t, ds.s) and dm.k1Inv == ds.k1Inv


def test_ch_workers_set_state_resume(sg, modulo):
    """set_state (cahn_hilliard.cpp:251-258) scatters both time levels onto
    the workers; stepping on is bitwise the one-GPU stepper's."""
    p = params(sg, 512, seed=5)
    single = sg.CHStepper(p)
    single.step_many(4)
    c, q = single.field(), single.previous_field()
    multi = sg.CHStepper(p, 1, 4)
    multi.set_state(c, q)
    assert multi.step_index() == 0
    single.step_many(5)
    multi.step_many(5)
    assert bits_equal(multi.field().values, single.field().values)
    assert bits_equal(multi.previous_field().values, single.previous_field().values)


def test_ch_workers_run_with_sink(sg, modulo):
    """run(params, numTiles, numWorkers, sink) with numWorkers = 4 emits the
    same diagnostics rows as the one-GPU run."""
    p = params(sg, 256, T=0.0)
    p.T = 20 * p.dt
    rows = {1: [], 4: []}
    for w in (1, 4):
        sink = sg.RunSink(diagEvery=5, onDiagnostics=lambda d, w=w: rows[w].append((d.t, d.s, d.k1Inv)))
        sg.run(p, 1, w, sink)
    assert rows[1] and rows[1] == rows[4]
