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

mode="p2p" fuses every exchange into a kernel (sg_chd_*_p2p): every
finished backward stage of a sweep is TMA-stored straight into the buffer of
the rank that consumes it (CUDA IPC-mapped peer memory over NVLink), so the
all-to-alls overlap the recurrence; the Woodbury corrections move to the
consumers (the y-sweep's load, the combine); the combine also stores the
halo rows of C^{n+1} into the neighbours' slabs. Steps 1, 3 and 5 become
barriers (a one-element NCCL all-reduce on the compute stream); only the
first step exchanges halos. Falls back to mode "nccl" when the geometry
does not allow it (sg_chd_set_peers).
"""
from __future__ import annotations

import ctypes as C

from . import _lib
from ._lib import InvalidArgument, check
from .slab import Slab, exchange_halos

HALO = 2


class DistCHStepper:
    def __init__(self, params, world: int = 1, rank: int = 0, dist=None, device="cuda", transport=None,
                 mode: str = "nccl"):
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
        self.mode = "nccl"
        if mode == "p2p":
            bufs = [C.c_void_p() for _ in range(4)]
            check(_lib.lib().sg_chd_p2p_buffers(self._h, *[C.byref(b) for b in bufs]))
            # recvX, recvY, y4xAll, y4yAll, then the two time-level ext slabs
            # (cur, prev at construction), whose halo rows the neighbours'
            # combines write
            self.p2p_buffers = [b.value for b in bufs] + [self.cur.data_ptr(), self.prev.data_ptr()]
            self._prev_idx = 1  # construction index of the buffer holding C^{n-1}
            self._halos_valid = False
            if transport is not None:
                transport.register(self)  # peers are wired once every rank exists
            elif world == 1:
                self.set_peers([[b] for b in self.p2p_buffers])
                self._flag = None
            else:
                self._ipc_peers()

    # -- P2P wiring
    def set_peers(self, tables):
        """tables: for each of (recvX, recvY, y4xAll, y4yAll, ext0, ext1) the
        device pointers of every rank, in rank order."""
        self._ext_tables = tables[4:6]
        arrs = [(C.c_void_p * self.world)(*t) for t in tables[:4]]
        ok = C.c_int()
        check(_lib.lib().sg_chd_set_peers(self._h, *arrs, C.byref(ok)))
        self.mode = "p2p" if ok.value else "nccl"
        return self.mode == "p2p"

    def _ipc_peers(self):
        """Exchange CUDA IPC handles of the four receive buffers (all_gather
        over the process group) and map the peers' buffers."""
        get_handle, open_handle, self._opened = ipc_handle_functions()
        tables, _ = exchange_peer_tables(self.dist, self.rank, self.world, self.p2p_buffers,
                                                    get_handle, open_handle)
        ok = self.set_peers(tables)
        flags = self.torch.tensor([1.0 if ok else 0.0],
                                  device=self.cur.device if self.dist.get_backend() == "nccl" else "cpu")
        self.dist.all_reduce(flags, op=self.dist.ReduceOp.MIN)
        if flags.item() < 1.0:  # every rank must take the same path
            self.mode = "nccl"
        self._flag = self.torch.zeros(1, device=self.cur.device)

    def _barrier(self):
        """Orders the peers' P2P writes before this rank reads them: each
        rank's all-reduce contribution is queued after its sweep kernel
        (NCCL). Over gloo (ranks sharing a GPU in tests): a device sync and a
        host barrier."""
        if self.transport is None and self.world > 1:
            if self.dist.get_backend() == "nccl":
                self.dist.all_reduce(self._flag)
            else:
                self.torch.cuda.current_stream().synchronize()
                self.dist.barrier()

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
        if self.mode == "p2p":
            if self._halos_valid:
                self._barrier()  # the neighbours' combines forwarded this step's halos
            else:
                self._halos()  # once: later halos arrive with the combine
                self._halos_valid = True
            check(_lib.lib().sg_chd_phase_x_p2p(self._h, self._p(self.cur), self._p(self.prev), self._s()))
            return
        self._halos()
        check(_lib.lib().sg_chd_phase_x(self._h, self._p(self.cur), self._p(self.prev), self._p(self.send), self._s()))

    def phase_y(self):
        if self.mode == "p2p":
            self._barrier()
            check(_lib.lib().sg_chd_phase_y_p2p(self._h, self._s()))
            return
        self._alltoall(self.ycol, self.send, 0)
        check(_lib.lib().sg_chd_phase_y(self._h, self._p(self.ycol), self._s()))

    def phase_combine(self):
        if self.mode == "p2p":
            self._barrier()
            up, dn = (self.rank - 1) % self.world, (self.rank + 1) % self.world
            ext = self._ext_tables[self._prev_idx]
            check(_lib.lib().sg_chd_combine_p2p(self._h, self._p(self.cur), self._p(self.prev), C.c_void_p(ext[up]),
                                                C.c_void_p(ext[dn]), self._s()))
            self._prev_idx ^= 1
        else:
            self._alltoall(self.recv, self.ycol, 1)
            check(_lib.lib().sg_chd_combine(self._h, self._p(self.cur), self._p(self.prev), self._p(self.recv),
                                            self._s()))
        self.cur, self.prev = self.prev, self.cur
        self.steps_done += 1

    def step(self):
        """One step. In P2P mode with graphs enabled (default at world = 1;
        opt-in via use_graphs for world > 1, where the barriers are NCCL
        all-reduces inside the capture) every step after the first replays
        a CUDA graph of the whole step — one per buffer parity, captured on
        first use — so the host issues one launch per step."""
        if self.mode == "p2p" and self._halos_valid and self._graphs_on():
            key = self._prev_idx
            g = self._graphs.get(key)
            if g is None:
                g = self.torch.cuda.CUDAGraph()
                with self.torch.cuda.graph(g):
                    self._step_body()  # records; the Python state advances as one step
                self._graphs[key] = g
            else:
                self._advance()
            g.replay()
            return
        self._step_body()

    def _step_body(self):
        self.phase_x()
        self.phase_y()
        self.phase_combine()

    def _advance(self):
        # the bookkeeping _step_body does (a replayed graph skips it)
        self.cur, self.prev = self.prev, self.cur
        self._prev_idx ^= 1
        self.steps_done += 1

    use_graphs = None  # None: on at world == 1 without a test transport

    def _graphs_on(self):
        if not hasattr(self, "_graphs"):
            self._graphs = {}
        if self.use_graphs is None:
            return self.world == 1 and self.transport is None
        return bool(self.use_graphs)

    def own_rows(self, which=0):
        """View of this rank's rows of C^n (which=0) or C^{n-1} (which=1)."""
        t = self.cur if which == 0 else self.prev
        return t[HALO:HALO + self.own]

    def __del__(self):
        try:
            for ptr in getattr(self, "_opened", []):
                _lib.lib().sg_ipc_close(C.c_void_p(ptr))
            if self._h.value:
                _lib.lib().sg_chd_destroy(C.byref(self._h))
        except Exception:
            pass


def ipc_handle_functions():
    """(get_handle, open_handle, bases) over the C ABI's CUDA IPC calls. A
    handle is the 64-byte IPC handle of the allocation plus the pointer's
    offset in it; opening maps the peer's allocation (its base is appended
    to `bases`, for sg_ipc_close) and re-applies the offset."""
    bases = []
    mapped = {}  # allocation handle -> mapped base: an allocation is opened once per process

    def get_handle(ptr):
        h = (C.c_char * 64)()
        off = C.c_size_t()
        check(_lib.lib().sg_ipc_get_handle(C.c_void_p(ptr), h, C.byref(off)))
        return bytes(h) + off.value.to_bytes(8, "little")

    def open_handle(hb):
        key = bytes(hb[:64])
        if key not in mapped:  # two buffers in one peer allocation share the mapping
            ptr = C.c_void_p()
            check(_lib.lib().sg_ipc_open_handle((C.c_char * 64).from_buffer_copy(hb[:64]), C.byref(ptr)))
            bases.append(ptr.value)
            mapped[key] = ptr.value
        return mapped[key] + int.from_bytes(hb[64:72], "little")

    return get_handle, open_handle, bases


def exchange_peer_tables(dist, rank, world, local_ptrs, get_handle, open_handle):
    """All-gather the IPC handles of every rank's receive buffers and map
    the peers' ones. Returns (tables, opened): tables[k][r] is buffer k of
    rank r as a pointer valid in this process (this rank's own pointers for
    r == rank), opened the pointers to close at teardown."""
    handles = [get_handle(p) for p in local_ptrs]
    gathered = [None] * world
    dist.all_gather_object(gathered, handles)
    tables = [[0] * world for _ in local_ptrs]
    opened = []
    for r in range(world):
        for k in range(len(local_ptrs)):
            if r == rank:
                tables[k][r] = local_ptrs[k]
            else:
                tables[k][r] = open_handle(gathered[r][k])
                opened.append(tables[k][r])
    return tables, opened


class LocalTransport:
    """In-process stand-in for NCCL when G ranks are simulated on one device
    (tests): halos and all-to-all blocks are copied between the ranks'
    buffers with exactly the layouts the collectives produce."""

    def __init__(self, ranks):
        self.ranks = ranks  # list of DistCHStepper, index = rank
        self.pending = {}
        self.p2p = []

    def register(self, st):
        """P2P mode: once all G ranks exist, give each every rank's receive
        buffers (the simulated 'peer memory' is the other ranks' buffers on
        the same device)."""
        self.p2p.append(st)
        if len(self.p2p) == st.world:
            tables = [[r.p2p_buffers[k] for r in sorted(self.p2p, key=lambda x: x.rank)] for k in range(6)]
            for r in self.p2p:
                r.set_peers(tables)

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
