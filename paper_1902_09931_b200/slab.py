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

import json
import os
import statistics
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

    def own_view(self, buf):
        t = self.slab.top
        return buf[t:t + self.slab.own]

    def apply(self, stream=None):
        """out(own rows of b) = stencil(a); returns after enqueueing."""
        from .stencil import launch_slab
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


def bench_multi_gpu(args, rank, world, local_rank, metric, unit, workload, peak, peak_kind):
    """Weak scaling: every rank owns a 32768 x 32768 slab of a periodic
    (world*32768) x 32768 grid; one step = halo exchange + application."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from . import _lib
    from .stencil import Extents, FunctionStencil
    if not dist.is_initialized():
        import os as _os
        _os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        _os.environ.setdefault("MASTER_PORT", "29511")
        _os.environ.setdefault("RANK", str(rank))
        _os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    nx = per = 32768
    ny = per * world
    slab = Slab(nx, ny, world, rank, 1, 1, True)
    kind = FunctionStencil(Extents(1, 1, 1, 1), "fn_weighted_3x3", list(np.random.default_rng(4).uniform(-1, 1, 9)))
    st = SlabStencil(slab, (1, 1, 1, 1), kind, torch.float64, f"cuda:{local_rank}", dist)
    g = torch.Generator(device="cuda").manual_seed(4 + rank)
    st.own_view(st.a).copy_(torch.rand((slab.own, nx), dtype=torch.float64, device="cuda", generator=g))
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        st.apply(stream.cuda_stream)
        st.swap()
    torch.cuda.synchronize()
    dist.barrier()
    l0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        st.apply(stream.cuda_stream)
        st.swap()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    launches = _lib.launch_count() - l0
    if rank == 0:
        value = nx * ny / (ms * 1e-3) / 1e9
        alg = nx * per * 16
        line = {"metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload + f", weak scaling: 32768x32768 y-slab per GPU ({nx}x{ny} total)",
                           "nx": nx, "ny": ny, "parallelism": f"y-slab x{world}, NCCL halo exchange",
                           "l2": "input 8 GiB per GPU >> L2"},
                "roofline": {"bound": "hbm", "achieved": alg / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                             "frac": alg / (ms * 1e-3) / 1e9 / peak, "traffic": None, "peak_kind": peak_kind,
                             "note": "per-GPU step time incl. halo exchange"},
                "gpu_launches": int(launches)}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
