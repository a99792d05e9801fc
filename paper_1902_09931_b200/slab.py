"""Multi-GPU y-slab domain decomposition for the stencil engine.

Replaces the reference's host tiling layer (make_tiles, grid.cpp:62-82, and
the WorkerPool fan-out, stencil.cpp:215-233) with a persistent decomposition:
one process per GPU (torchrun), each owning a contiguous block of rows
(ceil-first, exactly make_tiles' partition) stored with `top` halo rows
above and `bottom` halo rows below:

    ext buffer rows:  [ top halo | own rows (r1 - r0) | bottom halo ]

Per application, halo rows are exchanged with the ring neighbours over
torch.distributed point-to-point ops (NCCL over NVLink on the B200 box; gloo
in the CPU tests) while the interior rows — those whose windows stay inside
the slab — are computed on the compute stream; the boundary rows run after
the exchange lands. Periodic grids wrap rank 0 <-> rank G-1; non-periodic
grids leave the global frame untouched (stencil.cpp:35-38). Every output is
computed by the same kernel arithmetic as the single-GPU path, so results
are bitwise invariant in the GPU count.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


def make_tiles(ny: int, num_tiles: int):
    """Ceil-first contiguous row ranges (grid.cpp:62-82)."""
    if ny < 1:
        raise ValueError("make_tiles: ny must be >= 1")
    if num_tiles < 1 or num_tiles > ny:
        raise ValueError("make_tiles: numTiles must satisfy 1 <= numTiles <= ny")
    base, extra = divmod(ny, num_tiles)
    out, j = [], 0
    for t in range(num_tiles):
        rows = base + (1 if t < extra else 0)
        out.append((j, j + rows))
        j += rows
    return out


@dataclass
class Slab:
    nx: int
    ny: int
    world: int
    rank: int
    top: int
    bottom: int
    periodic: bool
    r0: int = 0
    r1: int = 0

    def __post_init__(self):
        self.r0, self.r1 = make_tiles(self.ny, self.world)[self.rank]
        if self.world > 1 and self.own < max(self.top, self.bottom):
            raise ValueError("slab: every rank needs at least max(top, bottom) rows")

    @property
    def own(self) -> int:
        return self.r1 - self.r0

    @property
    def ext_rows(self) -> int:
        return self.top + self.own + self.bottom

    @property
    def up(self):
        if self.rank > 0:
            return self.rank - 1
        return self.world - 1 if self.periodic else None

    @property
    def down(self):
        if self.rank < self.world - 1:
            return self.rank + 1
        return 0 if self.periodic else None

    def global_rows_of_ext(self):
        """Global row index held by each ext-buffer row (None = unused)."""
        rows = []
        for k in range(self.ext_rows):
            g = self.r0 - self.top + k
            if self.periodic:
                rows.append(g % self.ny)
            else:
                rows.append(g if 0 <= g < self.ny else None)
        return rows

    def output_rows(self):
        """Own rows to compute, in local output coordinates [a, b)."""
        a, b = 0, self.own
        if not self.periodic:
            a = max(a, self.top - self.r0)
            b = min(b, self.ny - self.bottom - self.r0)
        return a, max(a, b)

    def interior_rows(self):
        """Output rows whose windows need no halo row: [top, own - bottom)."""
        a, b = self.output_rows()
        return max(a, self.top), min(b, self.own - self.bottom)

    def desc(self, ext_cols, row0, row1):
        """sg_slab_desc for output rows [row0, row1) of this slab."""
        left, right = ext_cols
        if self.periodic:
            c0, c1 = 0, self.nx
        else:
            c0 = min(left, self.nx)
            c1 = max(min(self.nx - right, self.nx), c0)
        return dict(nx=self.nx, inRows=self.ext_rows, inShift=self.top, row0=row0, row1=row1,
                    col0=c0, col1=c1, wrapX=int(self.periodic), wrapY=0)


def exchange_ops(slab: Slab, ext, dist):
    """P2P ops filling the halo rows of `ext` (a (ext_rows, nx) tensor whose
    own rows are current). My top halo = the up neighbour's last `top` rows;
    my bottom halo = the down neighbour's first `bottom` rows."""
    top, bottom, own = slab.top, slab.bottom, slab.own
    ops = []
    if slab.world == 1:
        return ops
    if top and slab.up is not None:
        ops.append(dist.P2POp(dist.irecv, ext[0:top], slab.up))
    if bottom and slab.down is not None:
        ops.append(dist.P2POp(dist.irecv, ext[top + own:top + own + bottom], slab.down))
    if top and slab.down is not None:  # my last `top` rows are down's top halo
        ops.append(dist.P2POp(dist.isend, ext[own:top + own], slab.down))
    if bottom and slab.up is not None:  # my first `bottom` rows are up's bottom halo
        ops.append(dist.P2POp(dist.isend, ext[top:top + bottom], slab.up))
    return ops


def local_wrap_fill(slab: Slab, ext):
    """world == 1 periodic: the halos are the slab's own opposite rows."""
    if slab.world != 1 or not slab.periodic:
        return
    top, bottom, own = slab.top, slab.bottom, slab.own
    if top:
        ext[0:top].copy_(ext[own:own + top])
    if bottom:
        ext[top + own:top + own + bottom].copy_(ext[top:top + bottom])


def exchange_halos(slab: Slab, ext, dist=None):
    """Blocking halo exchange (setup, tests and the simple path). Over gloo,
    which has no CUDA send/recv, device slabs are staged through host
    copies."""
    if slab.world == 1:
        local_wrap_fill(slab, ext)
        return
    staged = None
    if getattr(ext, "is_cuda", False) and dist.get_backend() != "nccl":
        staged, ext = ext, ext.cpu()
    ops = exchange_ops(slab, ext, dist)
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    if staged is not None:
        top, own, bottom = slab.top, slab.own, slab.bottom
        if top:
            staged[0:top].copy_(ext[0:top])
        if bottom:
            staged[top + own:top + own + bottom].copy_(ext[top + own:top + own + bottom])


class SlabStencil:
    """One rank's share of a distributed stencil application.

    apply(): halo exchange (async NCCL) overlapped with the interior-row
    kernel, then the boundary-row kernels — all on the GPU through
    sg_stencil_launch."""

    def __init__(self, slab: Slab, ext, kind, dtype, device, dist=None):
        import torch
        from .stencil import Extents
        self.slab, self.kind, self.dist = slab, kind, dist
        self.ext = ext if isinstance(ext, Extents) else Extents(*ext)
        self.a = torch.zeros((slab.ext_rows, slab.nx), dtype=dtype, device=device)
        self.b = torch.zeros_like(self.a)
        self.torch = torch
        self.mode = "nccl"
        self._out = 1  # index of the output buffer in (a, b); swap() toggles it
        self._tables = None

    # -- P2P mode: the halo exchange fused into the stencil launch --------
    def p2p_buffers(self):
        """This rank's (a, b) ext buffers, to be exported to the neighbours."""
        return [self.a.data_ptr(), self.b.data_ptr()]

    def enable_p2p(self, tables, barrier=None):
        """tables[k][r]: rank r's buffer k (0 = a, 1 = b at construction) as
        a pointer valid in this process (IPC-mapped peer memory, or another
        simulated rank's buffer). From now on every apply() also stores the
        rows its neighbours need as halos straight into their output buffer
        (sg_stencil_launch_p2p), so no exchange precedes the next apply; the
        `barrier` (default: a one-element all-reduce on the compute stream
        when world > 1) orders those writes between applications. The
        caller fills the input's halos once before the first apply
        (exchange_halos)."""
        self._tables = tables
        self._barrier = barrier
        self.mode = "p2p"

    def _peers(self):
        s = self.slab
        esz = self.a.element_size()
        nx = s.nx
        up_ptr = dn_ptr = 0
        up_rows = dn_row0 = 0
        if s.up is not None and s.bottom:
            up = Slab(nx, s.ny, s.world, s.up, s.top, s.bottom, s.periodic)
            up_ptr = self._tables[self._out][s.up] + esz * (s.top + up.own) * nx  # its bottom halo
            up_rows = s.bottom  # my first `bottom` rows
        if s.down is not None and s.top:
            dn_ptr = self._tables[self._out][s.down]  # its top halo (ext rows 0..top)
            dn_row0 = s.own - s.top  # my last `top` rows
        return up_ptr, up_rows, dn_ptr, dn_row0

    def _apply_p2p(self, stream=None):
        from .stencil import launch_slab
        s = self.slab
        oa, ob = s.output_rows()
        if oa < ob:
            launch_slab(s.desc((self.ext.left, self.ext.right), oa, ob), self.ext, self.kind, self.a,
                        self.own_view(self.b), stream, peers=self._peers())
        if self._barrier is not None:
            self._barrier()
        elif s.world > 1:
            # the barrier must be ordered after THIS launch's peer stores: issue
            # it on the stream the kernel ran on, not torch's current stream
            with self.torch.cuda.stream(self._torch_stream(stream)):
                self.default_barrier()

    def default_barrier(self):
        """Orders every rank's peer stores before any rank's next read: a
        one-element NCCL all-reduce queued on the current stream (each
        rank's contribution follows its kernel), or, over gloo (ranks sharing
        a device in tests), a device sync + host barrier."""
        if self.dist.get_backend() == "nccl":
            if not hasattr(self, "_flag"):
                self._flag = self.torch.zeros(1, device=self.a.device)
            self.dist.all_reduce(self._flag)
        else:
            self.torch.cuda.current_stream().synchronize()
            self.dist.barrier()

    def _torch_stream(self, stream):
        torch = self.torch
        if stream is None:
            return torch.cuda.current_stream()
        if isinstance(stream, torch.cuda.Stream):
            return stream
        return torch.cuda.ExternalStream(int(stream))

    def own_view(self, buf):
        t = self.slab.top
        return buf[t:t + self.slab.own]

    def apply(self, stream=None):
        """out(own rows of b) = stencil(a); returns after enqueueing.

        NCCL form: the halo sends/receives are posted FIRST — the rows sent
        are own rows of `a`, complete once the previous application is — so
        the NCCL stream runs the exchange while the interior-row kernel
        (windows inside the slab) computes; the boundary-row kernels wait for
        the exchange. Everything is ordered on `stream` (default: torch's
        current stream)."""
        from .stencil import launch_slab
        if self.mode == "p2p":
            return self._apply_p2p(stream)
        s = self.slab
        lr = (self.ext.left, self.ext.right)
        out_own = self.own_view(self.b)
        ia, ib = s.interior_rows()
        oa, ob = s.output_rows()
        ts = self._torch_stream(stream)
        works = []
        if s.world > 1:
            ops = exchange_ops(s, self.a, self.dist)
            if ops:
                # ProcessGroupNCCL orders its stream after the CURRENT stream at
                # this point, i.e. after the previous application only
                with self.torch.cuda.stream(ts):
                    works = self.dist.batch_isend_irecv(ops)
        if ia < ib:
            launch_slab(s.desc(lr, ia, ib), self.ext, self.kind, self.a, out_own, ts.cuda_stream)
        if s.world == 1:
            with self.torch.cuda.stream(ts):
                local_wrap_fill(s, self.a)
        else:
            with self.torch.cuda.stream(ts):
                for r in works:
                    r.wait()  # makes `ts` wait on the NCCL stream
        if ia >= ib:
            if oa < ob:
                launch_slab(s.desc(lr, oa, ob), self.ext, self.kind, self.a, out_own, ts.cuda_stream)
            return
        if oa < ia:
            launch_slab(s.desc(lr, oa, ia), self.ext, self.kind, self.a, out_own, ts.cuda_stream)
        if ib < ob:
            launch_slab(s.desc(lr, ib, ob), self.ext, self.kind, self.a, out_own, ts.cuda_stream)

    def swap(self):
        self.a, self.b = self.b, self.a
        self._out ^= 1

    def apply_host(self, hin, hout, chunks: int = 0):
        """End-to-end application from/to pinned HOST memory.

        hin: (ext_rows, nx) host rows of the input in ext order — top halo,
        own rows, bottom halo (global rows `slab.global_rows_of_ext()`; rows
        outside a non-periodic grid are never read) — so a rank reading its
        share of a host-resident grid takes its halo rows from host memory
        and no device exchange is needed. hout: (own, nx) host output rows;
        outside the computed window (the non-periodic frame) it is left
        untouched, as the reference leaves its output frame (stencil.cpp:35-38).

        Pipelined in row chunks on three streams: the H2D of the ext rows
        chunk c+1 needs, the kernel on chunk c and the D2H of chunk c-1
        overlap (PCIe is full duplex). Same kernels and arithmetic as
        `apply` (bitwise equal); returns after the D2H copies complete."""
        from .stencil import launch_slab
        torch = self.torch
        s = self.slab
        H = s.top + s.bottom
        lr = (self.ext.left, self.ext.right)
        comp = torch.cuda.current_stream()
        if not hasattr(self, "_h2d"):
            self._h2d, self._d2h = torch.cuda.Stream(), torch.cuda.Stream()
        h2d, d2h = self._h2d, self._d2h
        if tuple(hin.shape) != (s.ext_rows, s.nx) or tuple(hout.shape) != (s.own, s.nx):
            raise ValueError("apply_host: hin must be (ext_rows, nx), hout (own, nx)")
        oa, ob = s.output_rows()
        if chunks <= 0:  # fill and drain cost one chunk each: many chunks (SG_SLAB_CHUNKS overrides)
            chunks = int(os.environ.get("SG_SLAB_CHUNKS", "64"))
        chunks = max(1, min(chunks, ob - oa))
        bounds = [(oa + (ob - oa) * c // chunks, oa + (ob - oa) * (c + 1) // chunks) for c in range(chunks)]
        desc0 = s.desc(lr, 0, 0)
        c0, c1 = desc0["col0"], desc0["col1"]
        full_rows = (c0, c1) == (0, s.nx)
        h2d.wait_stream(comp)  # the previous step's readers of `a` are done
        b_own = self.own_view(self.b)
        landed, done = [], []
        e0 = 0
        for c, (r0, r1) in enumerate(bounds):
            # output row j reads ext rows j .. j + H
            e1 = s.ext_rows if c == chunks - 1 else r1 + H
            with torch.cuda.stream(h2d):
                if e1 > e0:
                    self.a[e0:e1].copy_(hin[e0:e1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d)
            landed.append(ev)
            e0 = max(e0, e1)
        for c, (r0, r1) in enumerate(bounds):
            comp.wait_event(landed[c])
            if r0 < r1:
                launch_slab(s.desc(lr, r0, r1), self.ext, self.kind, self.a, b_own, comp.cuda_stream)
            ev = torch.cuda.Event()
            ev.record(comp)
            done.append(ev)
        with torch.cuda.stream(d2h):
            for c, (r0, r1) in enumerate(bounds):
                d2h.wait_event(done[c])
                if r0 >= r1:
                    continue
                if full_rows:
                    hout[r0:r1].copy_(b_own[r0:r1], non_blocking=True)
                else:
                    hout[r0:r1, c0:c1].copy_(b_own[r0:r1, c0:c1], non_blocking=True)
        d2h.synchronize()
        comp.wait_stream(d2h)

    def host_ext_rows(self, grid):
        """The (ext_rows, nx) rows apply_host reads, gathered from a full
        (ny, nx) host grid (rows outside a non-periodic grid are zero)."""
        import numpy as np
        rows = self.slab.global_rows_of_ext()
        out = np.zeros((len(rows), self.slab.nx), dtype=grid.dtype)
        for k, g in enumerate(rows):
            if g is not None:
                out[k] = grid[g]
        return out


def enable_p2p_ipc(st: SlabStencil, dist, fill_halos: bool = True) -> bool:
    """Production wiring of SlabStencil's P2P mode: exchange CUDA IPC
    handles of every rank's (a, b) buffers over the process group, map the
    peers' buffers, fill both buffers' halos once, and switch to the fused
    launch. Returns False (and stays in NCCL mode) if any rank cannot."""
    from .ch_dist import exchange_peer_tables, ipc_handle_functions

    get_handle, open_handle, st._opened = ipc_handle_functions()

    torch = st.torch
    ok = 1.0
    try:
        tables, _ = exchange_peer_tables(dist, st.slab.rank, st.slab.world, st.p2p_buffers(), get_handle,
                                         open_handle)
    except Exception:
        ok = 0.0
    flag = torch.tensor([ok], device=st.a.device if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if flag.item() < 1.0:
        return False
    if fill_halos:
        exchange_halos(st.slab, st.a, dist)
        exchange_halos(st.slab, st.b, dist)
    st.enable_p2p(tables)
    return True
