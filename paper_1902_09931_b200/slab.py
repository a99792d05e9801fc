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
import time
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
    """Blocking halo exchange (used by tests and the simple path)."""
    if slab.world == 1:
        local_wrap_fill(slab, ext)
        return
    ops = exchange_ops(slab, ext, dist)
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


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
            if not hasattr(self, "_flag"):
                self._flag = self.torch.zeros(1, device=self.a.device)
            self.dist.all_reduce(self._flag)

    def own_view(self, buf):
        t = self.slab.top
        return buf[t:t + self.slab.own]

    def apply(self, stream=None):
        """out(own rows of b) = stencil(a); returns after enqueueing."""
        from .stencil import launch_slab
        if self.mode == "p2p":
            return self._apply_p2p(stream)
        s = self.slab
        lr = (self.ext.left, self.ext.right)
        out_own = self.own_view(self.b)
        ia, ib = s.interior_rows()
        oa, ob = s.output_rows()
        if ia < ib:
            launch_slab(s.desc(lr, ia, ib), self.ext, self.kind, self.a, out_own, stream)
        if s.world == 1:
            local_wrap_fill(s, self.a)
        else:
            ops = exchange_ops(s, self.a, self.dist)
            if ops:
                for r in self.dist.batch_isend_irecv(ops):
                    r.wait()  # makes the current stream wait on the NCCL stream
        if ia >= ib:
            if oa < ob:
                launch_slab(s.desc(lr, oa, ob), self.ext, self.kind, self.a, out_own, stream)
            return
        if oa < ia:
            launch_slab(s.desc(lr, oa, ia), self.ext, self.kind, self.a, out_own, stream)
        if ib < ob:
            launch_slab(s.desc(lr, ib, ob), self.ext, self.kind, self.a, out_own, stream)

    def swap(self):
        self.a, self.b = self.b, self.a
        self._out ^= 1

    def apply_host(self, hin, hout, chunks: int = 0):
        """End-to-end application from/to pinned HOST memory: the own rows
        are uploaded in `chunks` row blocks on a copy stream (first and last
        block first, so the halo exchange can start early), each block's
        interior output rows are computed as soon as the block below has
        landed, and finished output blocks stream back on a second copy
        stream while later blocks compute. Same kernels and arithmetic as
        `apply` (bitwise equal); returns after the D2H copies complete."""
        from .stencil import launch_slab
        torch = self.torch
        s = self.slab
        own, top = s.own, s.top
        lr = (self.ext.left, self.ext.right)
        comp = torch.cuda.current_stream()
        if not hasattr(self, "_h2d"):
            self._h2d, self._d2h = torch.cuda.Stream(), torch.cuda.Stream()
        h2d, d2h = self._h2d, self._d2h
        if chunks <= 0:  # fill and drain cost one block each: many blocks (SG_SLAB_CHUNKS overrides)
            chunks = int(os.environ.get("SG_SLAB_CHUNKS", "64"))
        chunks = max(1, min(chunks, own))
        bounds = [(own * c // chunks, own * (c + 1) // chunks) for c in range(chunks)]
        order = [0, chunks - 1] + list(range(1, chunks - 1)) if chunks > 1 else [0]
        landed = {}
        h2d.wait_stream(comp)  # the previous step's readers of `a` are done
        a_own, b_own = self.own_view(self.a), self.own_view(self.b)
        for c in order:
            r0, r1 = bounds[c]
            with torch.cuda.stream(h2d):
                a_own[r0:r1].copy_(hin[r0:r1], non_blocking=True)
                landed[c] = torch.cuda.Event()
                landed[c].record(h2d)
        comp.wait_event(landed[0])
        comp.wait_event(landed[chunks - 1])
        if s.world == 1:
            local_wrap_fill(s, self.a)
            works = []
        else:
            ops = exchange_ops(s, self.a, self.dist)
            works = self.dist.batch_isend_irecv(ops) if ops else []
        ia, ib = s.interior_rows()
        oa, ob = s.output_rows()
        done = []
        for c in range(chunks):
            r0, r1 = bounds[c]
            if c + 1 < chunks:
                comp.wait_event(landed[c + 1])  # the window's bottom rows
            lo, hi = max(r0, ia), min(r1, ib)
            if lo < hi:
                launch_slab(s.desc(lr, lo, hi), self.ext, self.kind, self.a, b_own, comp.cuda_stream)
            ev = torch.cuda.Event()
            ev.record(comp)
            done.append(ev)
        for w in works:
            w.wait()
        edges = ((oa, ob),) if ia >= ib else ((oa, min(ia, ob)), (max(ib, oa), ob))
        for lo, hi in edges:
            if lo < hi:
                launch_slab(s.desc(lr, lo, hi), self.ext, self.kind, self.a, b_own, comp.cuda_stream)
        fin = torch.cuda.Event()
        fin.record(comp)
        # d2h is in-order: interior blocks first (each as soon as it is
        # computed), the blocks holding halo-dependent rows last
        edge = [bounds[c][0] < ia or bounds[c][1] > ib for c in range(chunks)]
        with torch.cuda.stream(d2h):
            for c in sorted(range(chunks), key=lambda c: edge[c]):
                r0, r1 = bounds[c]
                d2h.wait_event(fin if edge[c] else done[c])
                hout[r0:r1].copy_(b_own[r0:r1], non_blocking=True)
        d2h.synchronize()


def bench_multi_gpu(args, rank, world, local_rank, metric, unit, workload, peak, peak_kind, clocks_cls=None):
    """Weak scaling: every rank owns a 32768 x 32768 slab of a periodic
    (world*32768) x 32768 grid; one step = halo exchange + application.

    Returns rank 0's JSON line (None elsewhere). Device time is CUDA events
    on the compute stream, max over ranks; `e2e` adds, every step, the H2D
    copy of the rank's slab from pinned host memory and the D2H copy of its
    output rows (wall clock between barriers, max over ranks)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from . import _lib
    from .stencil import Extents, FunctionStencil
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    nx = per = 32768
    ny = per * world
    slab = Slab(nx, ny, world, rank, 1, 1, True)
    kind = FunctionStencil(Extents(1, 1, 1, 1), "fn_weighted_3x3", list(np.random.default_rng(4).uniform(-1, 1, 9)))
    st = SlabStencil(slab, (1, 1, 1, 1), kind, torch.float64, f"cuda:{local_rank}", dist)
    g = torch.Generator(device="cuda").manual_seed(4 + rank)
    st.own_view(st.a).copy_(torch.rand((slab.own, nx), dtype=torch.float64, device="cuda", generator=g))
    stream = torch.cuda.current_stream()
    halo = "NCCL halo exchange"
    if getattr(args, "halo", "nccl") == "p2p":
        torch.cuda.synchronize()
        if enable_p2p_ipc(st, dist):
            halo = "halo rows stored into the neighbours' buffers by the stencil kernel (P2P over NVLink)"

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        st.apply(stream.cuda_stream)
        st.swap()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    clk = clocks_cls(local_rank) if (clocks_cls is not None and rank == 0) else None
    if clk:
        clk.__enter__()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        st.apply(stream.cuda_stream)
        st.swap()
    e1.record()
    torch.cuda.synchronize()
    if clk:
        clk.__exit__(None, None, None)
    launches = _lib.launch_count() - l0
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    dist.barrier()

    e2e = None
    e2e_steps = getattr(args, "e2e_steps", 3)
    if not getattr(args, "skip_e2e", False) and e2e_steps > 0:
        try:  # 2 x 8.6 GB of pinned host memory per rank
            hin = torch.empty((slab.own, nx), dtype=torch.float64, pin_memory=True)
            hout = torch.empty_like(hin, pin_memory=True)
            ok = 1.0
        except RuntimeError:
            ok = 0.0
        t_ok = torch.tensor([ok], device="cuda")
        dist.all_reduce(t_ok, op=dist.ReduceOp.MIN)
        if t_ok.item() < 1.0:
            e2e_steps = 0
            e2e = {"error": "pinned host buffers (2 x 8.6 GB per rank) could not be allocated"}
    if not getattr(args, "skip_e2e", False) and e2e_steps > 0:
        hin.uniform_(-1, 1)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            st.apply_host(hin, hout)
        dt = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": nx * ny * e2e_steps / dt / 1e9, "unit": unit,
               "h2d_bytes_per_step": slab.own * nx * 8 * world, "d2h_bytes_per_step": slab.own * nx * 8 * world,
               "steps": e2e_steps,
               "path": "SlabStencil.apply_host on every rank: slab uploaded from / output downloaded to pinned host memory, row-chunk pipelined"}
    line = None
    if rank == 0:
        value = nx * ny / (ms * 1e-3) / 1e9
        alg = nx * per * 16
        line = {"metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload + f", weak scaling: 32768x32768 y-slab per GPU ({nx}x{ny} total)",
                           "nx": nx, "ny": ny, "parallelism": f"y-slab x{world}, {halo}",
                           "l2": "input 8 GiB per GPU >> L2"},
                "roofline": {"bound": "hbm", "achieved": alg / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                             "frac": alg / (ms * 1e-3) / 1e9 / peak, "traffic": None, "peak_kind": peak_kind,
                             "note": "per-GPU step time incl. halo exchange"},
                "gpu_launches": int(launches)}
        if clk:
            line["clocks"] = clk.summary()
        if e2e:
            line["e2e"] = e2e
    dist.destroy_process_group()
    return line


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
