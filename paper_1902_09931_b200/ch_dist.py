"""Distributed Cahn-Hilliard BDF2-ADI stepper: y-slabs over GPUs (config 5).

One process per GPU (torchrun, NCCL). Rank r owns rows [r*ny/G, (r+1)*ny/G)
of both time levels as "ext" slabs with 2 halo rows above and below. One
step (cahn_hilliard.cpp:260-328 across GPUs):

  1. halo exchange: 2 rows of C^n and C^{n-1} with the ring neighbours
     (the RHS reads a 5x5 window of Cbar = 2C^n - C^{n-1});
  2. sg_chd_phase_x: fused RHS kernel + x-sweep (rows are local systems) +
     Woodbury-corrected transpose, written PACKED as G blocks (own x nx/G);
  3. all-to-all #1: block q goes to rank q, which then holds columns
     [q*nx/G, (q+1)*nx/G) of every row — exactly the interleaved batch of the
     y-sweep (nx/G periodic systems of ny unknowns);
  4. sg_chd_phase_y: y-sweep with the Woodbury correction in place;
  5. all-to-all #2: back to row slabs (packed);
  6. sg_chd_combine: C^{n+1} = (2C^n - C^{n-1}) + v over C^{n-1}; swap roles.

Every arithmetic operation is the single-GPU step's, so C^n is bitwise
identical for every G (tests/test_ch_dist_gpu.py, tests/test_ch_dist.py).
"""
from __future__ import annotations

import ctypes as C

from . import _lib
from ._lib import InvalidArgument, check
from .slab import Slab, exchange_halos

HALO = 2


class DistCHStepper:
    def __init__(self, params, world: int = 1, rank: int = 0, dist=None, device="cuda", transport=None):
        import torch
        self.torch = torch
        self.p, self.world, self.rank, self.dist = params, world, rank, dist
        self.transport = transport  # test hook: in-process exchange for simulated ranks
        self._h = C.c_void_p()
        cp = params._c()
        check(_lib.lib().sg_chd_create(C.byref(cp), world, rank, C.byref(self._h)))
        own, nxq, r0 = C.c_int(), C.c_int(), C.c_int()
        check(_lib.lib().sg_chd_geometry(self._h, C.byref(own), C.byref(nxq), C.byref(r0)))
        self.own, self.nxq, self.r0 = own.value, nxq.value, r0.value
        nx, ny = params.nx, params.ny
        self.slab = Slab(nx, ny, world, rank, HALO, HALO, True)
        assert (self.slab.r0, self.slab.own) == (self.r0, self.own)
        dt = torch.float64
        self.cur = torch.zeros((self.own + 2 * HALO, nx), dtype=dt, device=device)
        self.prev = torch.zeros_like(self.cur)
        self.send = torch.empty(self.own * nx, dtype=dt, device=device)
        if world == 1 and transport is None:
            # one rank: both all-to-alls are the identity, so the three
            # buffers alias and no copy is made
            self.ycol = self.recv = self.send
        else:
            self.ycol = torch.empty(ny * self.nxq, dtype=dt, device=device)
            self.recv = torch.empty(self.own * nx, dtype=dt, device=device)
        self.steps_done = 0
        check(_lib.lib().sg_chd_init(self._h, self._p(self.cur), self._p(self.prev), self._s()))

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr())

    def _s(self):
        return C.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    # -- communication (NCCL in production; `transport` for simulated ranks)
    def _halos(self):
        if self.transport is not None:
            self.transport.halos(self)
            return
        exchange_halos(self.slab, self.cur, self.dist)
        exchange_halos(self.slab, self.prev, self.dist)

    def _alltoall(self, out, inp, phase):
        if self.transport is not None:
            self.transport.alltoall(self, out, inp, phase)
        elif self.world == 1:
            if out.data_ptr() != inp.data_ptr():
                out.copy_(inp)
        else:
            self.dist.all_to_all_single(out, inp)

    # -- the split step
    def phase_x(self):
        self._halos()
        check(_lib.lib().sg_chd_phase_x(self._h, self._p(self.cur), self._p(self.prev), self._p(self.send), self._s()))

    def phase_y(self):
        self._alltoall(self.ycol, self.send, 0)
        check(_lib.lib().sg_chd_phase_y(self._h, self._p(self.ycol), self._s()))

    def phase_combine(self):
        self._alltoall(self.recv, self.ycol, 1)
        check(_lib.lib().sg_chd_combine(self._h, self._p(self.cur), self._p(self.prev), self._p(self.recv), self._s()))
        self.cur, self.prev = self.prev, self.cur
        self.steps_done += 1

    def step(self):
        self.phase_x()
        self.phase_y()
        self.phase_combine()

    def own_rows(self, which=0):
        """View of this rank's rows of C^n (which=0) or C^{n-1} (which=1)."""
        t = self.cur if which == 0 else self.prev
        return t[HALO:HALO + self.own]

    def __del__(self):
        try:
            if self._h.value:
                _lib.lib().sg_chd_destroy(C.byref(self._h))
        except Exception:
            pass


class LocalTransport:
    """In-process stand-in for NCCL when G ranks are simulated on one device
    (tests): halos and all-to-all blocks are copied between the ranks'
    buffers with exactly the layouts the collectives produce."""

    def __init__(self, ranks):
        self.ranks = ranks  # list of DistCHStepper, index = rank
        self.pending = {}

    def halos(self, st):
        # fill st's halos from the neighbours' own rows (periodic ring)
        G = st.world
        for buf_name in ("cur", "prev"):
            ext = getattr(st, buf_name)
            up = self.ranks[(st.rank - 1) % G]
            dn = self.ranks[(st.rank + 1) % G]
            up_own = getattr(up, buf_name)[HALO:HALO + up.own]
            dn_own = getattr(dn, buf_name)[HALO:HALO + dn.own]
            ext[0:HALO].copy_(up_own[up.own - HALO:])
            ext[HALO + st.own:].copy_(dn_own[:HALO])

    def alltoall(self, st, out, inp, phase):
        # all ranks must have produced `inp` before anyone reads: the test
        # drives ranks phase by phase, so every rank's input is ready here
        G = st.world
        blk = out.numel() // G
        for q in range(G):
            src = getattr(self.ranks[q], "send" if phase == 0 else "ycol")
            out[q * blk:(q + 1) * blk].copy_(src[st.rank * blk:(st.rank + 1) * blk])
