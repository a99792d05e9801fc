"""GPU: the production P2P wiring across PROCESSES. Two ranks (spawned
processes, gloo for the host-side exchange) share the one GPU: each exports
CUDA IPC handles of its slab buffers (allocation handle + offset), maps the
other's, and the fused stencil launches store the halo rows into the peer
process's buffer. Three applications (barrier: device sync + gloo barrier)
must equal the single-grid result bitwise."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1902_09931_b200 as sg
        from paper_1902_09931_b200.slab import Slab, SlabStencil, enable_p2p_ipc
        sg._lib.check(sg._lib.lib().sg_init(0))
        nx, ny = 256, 64
        rng = np.random.default_rng(5)
        g = rng.uniform(-1, 1, (ny, nx))
        w = list(rng.uniform(-1, 1, 9))
        kind = sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", w)
        slab = Slab(nx, ny, world, rank, 1, 1, True)
        # a torch-allocated buffer at an offset inside its allocation tests
        # the (handle, offset) form
        pad = torch.zeros(1000, dtype=torch.float64, device="cuda")
        st = SlabStencil(slab, (1, 1, 1, 1), kind, torch.float64, "cuda")
        for k, gr in enumerate(slab.global_rows_of_ext()):
            st.a[k] = torch.from_numpy(g[gr])
        torch.cuda.synchronize()
        ok = enable_p2p_ipc(st, dist, fill_halos=False)
        if not ok:
            q.put((rank, "no-p2p"))
            return

        def barrier():
            torch.cuda.synchronize()
            dist.barrier()

        st._barrier = barrier
        for _ in range(3):
            st.apply()
            st.swap()
        torch.cuda.synchronize()
        got = st.own_view(st.a).cpu().numpy()
        want = g
        from oracle.oracle import Restatement
        orc = Restatement()
        for _ in range(3):
            want = orc.stencil(want, (1, 1, 1, 1), w, fn="fn_weighted_3x3")
        same = np.array_equal(got.view(np.uint64), want[slab.r0:slab.r1].view(np.uint64))
        del pad
        q.put((rank, "ok" if same else "mismatch"))
    except Exception as e:  # report, do not hang the other rank
        q.put((rank, "error: " + repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_halo_forwarding_across_processes(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


def _ch_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1902_09931_b200 as sg
        from paper_1902_09931_b200.ch_dist import HALO, DistCHStepper
        sg._lib.check(sg._lib.lib().sg_init(0))
        n = 256
        p = sg.CHParams(nx=n, ny=n)
        p.dt = 0.1 * p.dx()
        p.T = 1.0
        st = DistCHStepper(p, world, rank, dist, mode="p2p")
        if st.mode != "p2p":
            q.put((rank, "no-p2p"))
            return

        def barrier():
            torch.cuda.synchronize()
            dist.barrier()

        def halos():  # first step only: through the host (gloo has no CUDA P2P)
            for buf in (st.cur, st.prev):
                own = buf[HALO:HALO + st.own].cpu()
                parts = [torch.empty_like(own) for _ in range(world)]
                dist.all_gather(parts, own)
                full = torch.cat(parts)
                rows = [(st.r0 - HALO + k) % n for k in range(st.own + 2 * HALO)]
                buf.copy_(full[rows].to(buf.device))

        st._barrier = barrier
        st._halos = halos
        steps = 4
        for _ in range(steps):
            st.step()
        torch.cuda.synchronize()
        single = sg.CHStepper(p)
        single.step_many(steps)
        want = single.field().values[st.r0:st.r0 + st.own]
        got = st.own_rows(0).cpu().numpy()
        q.put((rank, "ok" if np.array_equal(got.view(np.uint64), want.view(np.uint64)) else "mismatch"))
    except Exception as e:
        q.put((rank, "error: " + repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_ch_p2p_across_processes(world):
    """The distributed CH P2P step across processes on one GPU: IPC-mapped
    receive buffers written by the sweeps' TMA stores and the combine's halo
    forwarding of the other process — bitwise equal to the single-GPU
    stepper after 4 steps."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ch_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res
