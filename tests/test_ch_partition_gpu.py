"""Opt-in partitioned (SPIKE-type) CH sweeps (sg_ch_set_partition): P
segments per system solved as independent chains plus a 4P x 4P interface
system. Not bitwise — the bar is the north star's CH tolerance, 1e-9
relative L2 after 100 steps, against the bitwise path (itself bitwise equal
to the unmodified reference CHStepper, tests/test_ch_gpu.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run(sg, n, steps, P):
    p = sg.CHParams(nx=n, ny=n)
    p.dt = 0.1 * p.dx()
    p.T = steps * p.dt
    st = sg.CHStepper(p)
    if P:
        st.set_partition(P)
    st.step_many(steps)
    st.synchronize()
    return st.field().values.copy(), st.previous_field().values.copy()


@pytest.mark.parametrize("n,P", [(256, 2), (256, 4), (512, 8), (1024, 4), (1024, 16)])
def test_partitioned_within_north_star_after_100_steps(sg, n, P):
    c0, p0 = run(sg, n, 100, 0)
    c1, p1 = run(sg, n, 100, P)
    assert rel_l2(c1, c0) <= 1e-9 and rel_l2(p1, p0) <= 1e-9


def test_partition_off_is_bitwise_again(sg):
    p = sg.CHParams(nx=256, ny=256)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    a = sg.CHStepper(p)
    a.set_partition(4)
    a.step_many(3)
    a.set_partition(0)
    a.step_many(5)
    b = sg.CHStepper(p)
    b.set_partition(4)
    b.step_many(3)
    b.synchronize()
    b.set_partition(1)
    b.step_many(5)
    assert np.array_equal(a.field().values.view(np.uint64), b.field().values.view(np.uint64))


def test_partition_single_mode_matches_analytic_symbol(sg):
    """test_cahn_hilliard.cpp:292-318's oracle for the GPU ADI step: a
    single Fourier mode (nonlinearity off) evolves by the rational symbol of
    the scheme; 10 steps within 1e-12, partitioned too."""
    n = 256
    p = sg.CHParams(nx=n, ny=n)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    p.nonlinearEnabled = False
    x = np.arange(n) * p.dx()
    f = np.cos(3 * x)[None, :] * np.cos(2 * x)[:, None] * 0.1
    ref = sg.CHStepper(p)
    g = sg.Grid2D.from_array(f.copy())
    ref.set_state(g, g)
    ref.step_many(10)
    part = sg.CHStepper(p)
    part.set_partition(4)
    part.set_state(g, g)
    part.step_many(10)
    assert rel_l2(part.field().values, ref.field().values) <= 1e-12


def test_partition_rejects_bad_segments(sg):
    p = sg.CHParams(nx=256, ny=256)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    st = sg.CHStepper(p)
    with pytest.raises(sg.InvalidArgument):
        st.set_partition(3)  # 256 / 3 is not a whole number of 64-row stages
    with pytest.raises(sg.InvalidArgument):
        st.set_partition(17)


def test_partition_is_single_gpu_only(sg):
    """numWorkers > 1 steppers (config 5's distributed step) keep the bitwise
    sweeps: the partitioned mode is rejected there (at 8192^2
    any reordering exceeds the 1e-9 bar)."""
    p = sg.CHParams(nx=256, ny=256)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    old = sg.get_device_map()
    sg.set_device_map("modulo")
    try:
        st = sg.CHStepper(p, 1, 2)
        assert st.workers()[0] == 2
        with pytest.raises(sg.InvalidArgument):
            st.set_partition(4)
    finally:
        sg.set_device_map(old)
