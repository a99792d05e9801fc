"""GPU: the distributed CH step (y-slabs + two all-to-all transposes, config
5's algorithm) is bitwise identical to the single-GPU stepper and to the
oracle for every world size. Ranks are simulated on one device with the
in-process LocalTransport, which moves exactly the blocks NCCL would."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                                                 np.ascontiguousarray(b).view(np.uint64))


def params(sg, nx, ny, **kw):
    p = sg.CHParams(nx=nx, ny=ny)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    for k, v in kw.items():
        setattr(p, k, v)
    return p


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("nx,ny", [(64, 64), (128, 32), (32, 128)])
def test_distributed_ch_bitwise(sg, orc, G, nx, ny):
    import torch
    from paper_1902_09931_b200.ch_dist import DistCHStepper, LocalTransport
    if ny // G < 2 or nx % G:
        pytest.skip("slab too thin")
    p = params(sg, nx, ny, seed=7)
    ranks = []
    tr = LocalTransport(ranks)
    for r in range(G):
        ranks.append(DistCHStepper(p, G, r, transport=tr))
    steps = 6
    for _ in range(steps):
        for st in ranks:
            st.phase_x()
        for st in ranks:
            st.phase_y()
        for st in ranks:
            st.phase_combine()
    torch.cuda.synchronize()
    got = np.concatenate([st.own_rows(0).cpu().numpy() for st in ranks], axis=0)
    got_prev = np.concatenate([st.own_rows(1).cpu().numpy() for st in ranks], axis=0)
    single = sg.CHStepper(p)
    single.step_many(steps)
    assert bits_equal(got, single.field().values)
    assert bits_equal(got_prev, single.previous_field().values)
    c0 = orc.ch_initial_condition(nx, ny, seed=7)
    want, _ = orc.ch_run(dict(D=p.D, gamma=p.gamma, lx=p.lx, ly=p.ly, dt=p.dt, nx=nx, ny=ny), steps, c0, c0)
    assert bits_equal(got, want)


def test_distributed_ch_validation(sg):
    from paper_1902_09931_b200.ch_dist import DistCHStepper
    with pytest.raises(sg.InvalidArgument):
        DistCHStepper(params(sg, 64, 64), 3, 0)  # 3 does not divide 64
    with pytest.raises(sg.InvalidArgument):
        DistCHStepper(params(sg, 64, 64), 64, 0)  # 1 row per rank < 2-row halo


@pytest.mark.parametrize("G,nx,ny", [(1, 256, 256), (2, 256, 256), (2, 512, 256), (4, 512, 512), (8, 1024, 1024)])
def test_distributed_ch_p2p_bitwise(sg, G, nx, ny):
    """The P2P step (both all-to-alls fused into the sweeps' TMA stores into
    the consumers' buffers, corrections applied by the consumers) is bitwise
    identical to the single-GPU stepper. Simulated ranks: the 'peer memory'
    each sweep stores into is the other ranks' buffers on this device."""
    import torch
    from paper_1902_09931_b200.ch_dist import DistCHStepper, LocalTransport
    p = params(sg, nx, ny, seed=11)
    ranks = []
    tr = LocalTransport(ranks)
    for r in range(G):
        ranks.append(DistCHStepper(p, G, r, transport=tr, mode="p2p"))
    assert all(st.mode == "p2p" for st in ranks)
    steps = 5
    for _ in range(steps):
        for st in ranks:
            st.phase_x()
        for st in ranks:
            st.phase_y()
        for st in ranks:
            st.phase_combine()
    torch.cuda.synchronize()
    got = np.concatenate([st.own_rows(0).cpu().numpy() for st in ranks], axis=0)
    got_prev = np.concatenate([st.own_rows(1).cpu().numpy() for st in ranks], axis=0)
    single = sg.CHStepper(p)
    single.step_many(steps)
    assert bits_equal(got, single.field().values)
    assert bits_equal(got_prev, single.previous_field().values)


def test_distributed_ch_p2p_falls_back_when_tiles_do_not_fit(sg):
    """own = 32 rows is not a multiple of the sweep stage: the P2P wiring
    reports the path unavailable and the stepper keeps the NCCL form."""
    from paper_1902_09931_b200.ch_dist import DistCHStepper, LocalTransport
    p = params(sg, 64, 64)
    ranks = []
    tr = LocalTransport(ranks)
    for r in range(2):
        ranks.append(DistCHStepper(p, 2, r, transport=tr, mode="p2p"))
    assert all(st.mode == "nccl" for st in ranks)


def test_distributed_ch_p2p_graph_replay_world1(sg):
    """World 1, P2P mode: steps after the first replay per-parity CUDA graphs
    of the whole step (halo forwarding included) — bitwise equal to the
    single-GPU stepper, both time levels, odd and even step counts."""
    import torch
    from paper_1902_09931_b200.ch_dist import DistCHStepper
    p = params(sg, 256, 256, seed=13)
    st = DistCHStepper(p, 1, 0, mode="p2p")
    assert st.mode == "p2p"
    single = sg.CHStepper(p)
    for steps in (1, 2, 5):
        for _ in range(steps):
            st.step()
        single.step_many(steps)
        torch.cuda.synchronize()
        assert bits_equal(st.own_rows(0).cpu().numpy(), single.field().values)
        assert bits_equal(st.own_rows(1).cpu().numpy(), single.previous_field().values)
    assert len(st._graphs) == 2
