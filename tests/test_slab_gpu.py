"""GPU: the y-slab path computes exactly the single-GPU result.

Simulates G ranks on one device: each slab's extended buffer is filled by
the same halo plan the distributed path uses (rows looked up from the
global grid by Slab.global_rows_of_ext, which tests/test_slab_dist.py proves
equal to what the gloo/NCCL exchange delivers), the slab kernels run
through sg_stencil_launch (interior rows + boundary rows, as SlabStencil
does), and the concatenated output must equal the full-grid oracle BITWISE
for every G (bitwise invariance in the GPU count)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("ext,periodic,fn", [((1, 1, 1, 1), True, "fn_weighted_3x3"),
                                             ((1, 1, 1, 1), False, "weights"),
                                             ((2, 2, 2, 2), True, "weights"),
                                             ((0, 0, 1, 2), False, "weights"),
                                             ((2, 2, 0, 0), False, "weights")])
def test_slabs_equal_full_grid(sg, orc, G, ext, periodic, fn):
    import torch
    from paper_1902_09931_b200.slab import Slab, SlabStencil
    rng = np.random.default_rng(G * 7 + ext[0])
    nx, ny = 192, 64
    g = rng.uniform(-1, 1, (ny, nx))
    W = (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
    w = list(rng.uniform(-2, 2, 9 if fn != "weights" else W))
    e = sg.Extents(*ext)
    kind = sg.WeightStencil(e, w) if fn == "weights" else sg.FunctionStencil(e, fn, w)
    sentinel = -12345.678
    want = orc.stencil(g, ext, w, periodic=periodic, fn=fn, out=np.full_like(g, sentinel))
    got = np.full_like(g, sentinel)
    for r in range(G):
        slab = Slab(nx, ny, G, r, ext[2], ext[3], periodic)
        st = SlabStencil(slab, e, kind, torch.float64, "cuda")
        rows = slab.global_rows_of_ext()
        for k, gr in enumerate(rows):
            if gr is not None:
                st.a[k] = torch.from_numpy(g[gr])
        st.own_view(st.b).copy_(torch.from_numpy(got[slab.r0:slab.r1]))
        # halos already in place: run the same kernel split as SlabStencil.apply
        from paper_1902_09931_b200.stencil import launch_slab
        lr = (e.left, e.right)
        out_own = st.own_view(st.b)
        ia, ib = slab.interior_rows()
        oa, ob = slab.output_rows()
        spans = [(ia, ib), (oa, min(ia, ob)), (max(ib, oa), ob)] if ia < ib else [(oa, ob)]
        for a_, b_ in spans:
            if a_ < b_:
                launch_slab(slab.desc(lr, a_, b_), e, kind, st.a, out_own)
        torch.cuda.synchronize()
        got[slab.r0:slab.r1] = out_own.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_slab_stencil_apply_single_rank_periodic(sg, orc):
    """SlabStencil.apply() end to end with world = 1 (local wrap fill)."""
    import torch
    from paper_1902_09931_b200.slab import Slab, SlabStencil
    rng = np.random.default_rng(3)
    g = rng.uniform(-1, 1, (40, 128))
    w = list(rng.uniform(-1, 1, 9))
    kind = sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", w)
    slab = Slab(128, 40, 1, 0, 1, 1, True)
    st = SlabStencil(slab, (1, 1, 1, 1), kind, torch.float64, "cuda")
    st.own_view(st.a).copy_(torch.from_numpy(g))
    for _ in range(3):
        st.apply()
        st.swap()
    torch.cuda.synchronize()
    want = g
    for _ in range(3):
        want = orc.stencil(want, (1, 1, 1, 1), w, fn="fn_weighted_3x3")
    assert np.array_equal(st.own_view(st.a).cpu().numpy().view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("ext,periodic,chunks", [((1, 1, 1, 1), True, 4), ((2, 2, 2, 2), True, 7),
                                                 ((1, 1, 1, 1), False, 5), ((0, 0, 1, 2), False, 1)])
def test_apply_host_pipeline_equals_oracle(sg, orc, ext, periodic, chunks):
    """SlabStencil.apply_host (pinned host in/out, row-chunk pipelined
    H2D / compute / D2H — the e2e path of bench.py --slab) is bitwise equal
    to the oracle, repeated so buffer reuse across steps is exercised."""
    import torch
    from paper_1902_09931_b200.slab import Slab, SlabStencil
    rng = np.random.default_rng(11)
    nx, ny = 256, 96
    W = (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
    w = list(rng.uniform(-2, 2, W))
    kind = sg.WeightStencil(sg.Extents(*ext), w)
    slab = Slab(nx, ny, 1, 0, ext[2], ext[3], periodic)
    st = SlabStencil(slab, ext, kind, torch.float64, "cuda")
    sentinel = -12345.678
    st.own_view(st.b).fill_(sentinel)
    hin = torch.empty((slab.ext_rows, nx), dtype=torch.float64, pin_memory=True)
    hout = torch.full((ny, nx), sentinel, dtype=torch.float64, pin_memory=True)
    for rep in range(2):
        g = rng.uniform(-1, 1, (ny, nx))
        hin.copy_(torch.from_numpy(st.host_ext_rows(g)))
        st.apply_host(hin, hout, chunks=chunks)
        want = orc.stencil(g, ext, w, periodic=periodic, out=np.full_like(g, sentinel))
        assert np.array_equal(hout.numpy().view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("G", [1, 2, 3, 4])
@pytest.mark.parametrize("ext,periodic,fn", [((1, 1, 1, 1), True, "fn_weighted_3x3"),
                                             ((2, 2, 2, 2), True, "weights"),
                                             ((1, 1, 1, 1), False, "weights"),
                                             ((0, 0, 1, 2), False, "weights")])
def test_p2p_fused_halo_steps_equal_full_grid(sg, orc, G, ext, periodic, fn):
    """P2P mode: each application also stores the rows the neighbours need
    straight into their output buffers' halo rows (sg_stencil_launch_p2p) —
    no exchange between applications. Simulated ranks on one device (the
    'peer memory' is the other ranks' buffers); 3 applications with swaps
    equal the full-grid oracle BITWISE for every G, frames included."""
    import torch
    from paper_1902_09931_b200.slab import Slab, SlabStencil
    rng = np.random.default_rng(G * 11 + ext[2])
    nx, ny = 128, 48
    g = rng.uniform(-1, 1, (ny, nx))
    W = (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
    w = list(rng.uniform(-2, 2, 9 if fn != "weights" else W))
    e = sg.Extents(*ext)
    kind = sg.WeightStencil(e, w) if fn == "weights" else sg.FunctionStencil(e, fn, w)
    sentinel = -12345.678
    A, B = g.copy(), np.full_like(g, sentinel)
    for _ in range(3):
        B = orc.stencil(A, ext, w, periodic=periodic, fn=fn, out=B)
        A, B = B, A
    ranks = []
    for r in range(G):
        slab = Slab(nx, ny, G, r, ext[2], ext[3], periodic)
        st = SlabStencil(slab, e, kind, torch.float64, "cuda")
        for buf, src in ((st.a, g), (st.b, np.full_like(g, sentinel))):
            for k, gr in enumerate(slab.global_rows_of_ext()):  # own rows + initial halos
                if gr is not None:
                    buf[k] = torch.from_numpy(src[gr])
        ranks.append(st)
    tables = [[st.p2p_buffers()[k] for st in ranks] for k in range(2)]
    for st in ranks:
        st.enable_p2p(tables, barrier=lambda: None)
    for _ in range(3):
        for st in ranks:  # one stream: every rank's writes land before the next application
            st.apply()
        for st in ranks:
            st.swap()
    torch.cuda.synchronize()
    got = np.concatenate([st.own_view(st.a).cpu().numpy() for st in ranks], axis=0)
    assert np.array_equal(got.view(np.uint64), A.view(np.uint64))
