"""CPU multi-process tests of the y-slab decomposition (gloo backend).

Covers the host side of the N>1 path: the partition equals make_tiles'
(grid.cpp:62-82), and after the halo exchange every rank's extended slab
holds exactly the global rows its stencil windows read (periodic wrap
rank 0 <-> G-1; non-periodic frames). The compute on an extended slab is
covered on the GPU by tests/test_slab_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1902_09931_b200.slab import Slab, exchange_halos, make_tiles


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for nx, ny, top, bottom, periodic in cases:
            g = np.arange(nx * ny, dtype=np.float64).reshape(ny, nx) * 1.5 - 7.0
            slab = Slab(nx, ny, world, rank, top, bottom, periodic)
            ext = torch.full((slab.ext_rows, nx), float("nan"), dtype=torch.float64)
            ext[top:top + slab.own] = torch.from_numpy(g[slab.r0:slab.r1])
            exchange_halos(slab, ext, dist)
            for k, gr in enumerate(slab.global_rows_of_ext()):
                if gr is None:
                    continue
                if not torch.equal(ext[k], torch.from_numpy(g[gr])):
                    q.put((rank, "mismatch", nx, ny, top, bottom, periodic, k))
                    return
        q.put((rank, "ok"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_halo_exchange(world):
    cases = [(8, 12, 1, 1, True), (8, 12, 1, 1, False), (5, 9, 2, 1, True), (6, 10, 0, 2, True),
             (4, 7, 2, 2, False), (3, 6, 0, 0, True)]
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


def test_partition_matches_make_tiles_and_rows():
    for ny in range(1, 40):
        for world in range(1, min(ny, 9) + 1):
            tiles = make_tiles(ny, world)
            assert tiles[0][0] == 0 and tiles[-1][1] == ny
            for r in range(world):
                s = Slab(16, ny, world, r, 0, 0, True)
                assert (s.r0, s.r1) == tiles[r]
    s = Slab(16, 10, 3, 0, 1, 2, False)
    assert s.output_rows() == (1, 4) and s.interior_rows() == (1, 2)
    s = Slab(16, 10, 3, 2, 1, 2, False)
    assert s.output_rows() == (0, 1)
    with pytest.raises(ValueError):
        Slab(16, 4, 4, 0, 2, 2, True)


def _a2a_worker(rank, world, port, q):
    """The packed all-to-all layout of the distributed CH step
    (ch_dist.py): row slabs -> column slabs -> row slabs."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny = 12, 8 * world
        own, nxq = ny // world, nx // world
        g = np.arange(nx * ny, dtype=np.float64).reshape(ny, nx)
        mine = g[rank * own:(rank + 1) * own]
        # packed: block q = columns [q*nxq, (q+1)*nxq) of my rows
        send = torch.from_numpy(np.concatenate([mine[:, qq * nxq:(qq + 1) * nxq].ravel() for qq in range(world)]))
        ycol = torch.empty(ny * nxq, dtype=torch.float64)
        dist.all_to_all_single(ycol, send)
        ok = np.array_equal(ycol.numpy().reshape(ny, nxq), g[:, rank * nxq:(rank + 1) * nxq])
        back = torch.empty(own * nx, dtype=torch.float64)
        dist.all_to_all_single(back, ycol)
        ok = ok and np.array_equal(back.numpy(), send.numpy())
        q.put((rank, "ok" if ok else "bad"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_ch_alltoall_layout(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_a2a_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


def _p2p_worker(rank, world, port, q):
    """P2P wiring of the distributed CH step with fake pointers: the IPC
    handle of a 'buffer' encodes (rank, k); opening it must yield the peer's
    pointer, and every rank must see the same rank-ordered tables."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1902_09931_b200.ch_dist import exchange_peer_tables

        def ptr(r, k):
            return 0x10000000 * (r + 1) + 0x1000 * k

        local = [ptr(rank, k) for k in range(4)]
        get_handle = lambda p: p.to_bytes(8, "little") * 8  # a 64-byte "handle"
        opened_log = []

        def open_handle(hb):
            assert len(hb) == 64
            p = int.from_bytes(hb[:8], "little")
            opened_log.append(p)
            return p + 7  # a mapped alias differs from the exporter's pointer

        tables, opened = exchange_peer_tables(dist, rank, world, local, get_handle, open_handle)
        ok = all(tables[k][r] == (ptr(r, k) if r == rank else ptr(r, k) + 7)
                 for k in range(4) for r in range(world))
        ok = ok and sorted(opened) == sorted(p + 7 for p in opened_log) and len(opened) == 4 * (world - 1)
        q.put((rank, "ok" if ok else "bad"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ch_p2p_peer_tables(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res
