"""Small end-to-end workload over every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): stencils (TMA fast path FP64/FP32,
tall windows, non-periodic, generic; k_tma_g on asymmetric windows, odd
rows and misaligned bases), uniform and general penta solves, CH
steps (transposed-input sweeps, steady-state step, tail combine), the
distributed CH P2P step and the slab P2P halo forwarding on simulated ranks."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1902_09931_b200 as sg
from paper_1902_09931_b200.ch_dist import DistCHStepper, LocalTransport
from paper_1902_09931_b200.slab import Slab, SlabStencil

rng = np.random.default_rng(0)
sg._lib.check(sg._lib.lib().sg_init(0))
# stencils
for dt in (torch.float64, torch.float32):
    a = torch.rand((96, 256), dtype=dt, device="cuda")
    b = torch.zeros_like(a)
    for ext, mode, fn in [((1, 1, 1, 1), sg.BoundaryMode.Periodic, "fn_weighted_3x3"),
                          ((2, 2, 2, 2), sg.BoundaryMode.Periodic, None),
                          ((2, 2, 0, 0), sg.BoundaryMode.NonPeriodic, None),
                          ((1, 2, 0, 1), sg.BoundaryMode.NonPeriodic, None)]:
        e = sg.Extents(*ext)
        nv = (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
        kind = sg.FunctionStencil(e, fn, list(rng.uniform(-1, 1, 9))) if fn else sg.WeightStencil(e, list(rng.uniform(-1, 1, nv)))
        plan = sg.create_plan(sg.Direction.XY, mode, kind, a, b, 1, 1)
        sg.compute(plan)
        sg.destroy_plan(plan)
    # k_tma_g: asymmetric windows, odd rows (every 16 B phase), misaligned base
    for nx, off in ((97, 0), (2053, 1), (256, 1)):
        buf_a = torch.rand(41 * nx + 1, dtype=dt, device="cuda")
        buf_b = torch.zeros(41 * nx + 1, dtype=dt, device="cuda")
        a2, b2 = buf_a[off:off + 41 * nx].view(41, nx), buf_b[off:off + 41 * nx].view(41, nx)
        for ext, mode in [((3, 1, 0, 0), sg.BoundaryMode.Periodic), ((2, 1, 1, 2), sg.BoundaryMode.NonPeriodic),
                          ((1, 1, 1, 1), sg.BoundaryMode.Periodic), ((0, 8, 4, 4), sg.BoundaryMode.Periodic)]:
            nv = (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
            plan = sg.create_plan(sg.Direction.XY, mode, sg.WeightStencil(sg.Extents(*ext), list(rng.uniform(-1, 1, nv))),
                                  a2, b2, 1, 1)
            sg.compute(plan)
            sg.destroy_plan(plan)
# a window function registered from source (NVRTC-compiled kernels)
sg.register_function_source("san_fn", "return window[rowStride + 1] * coe[0] - window[0];")
for nx in (256, 97):
    a3 = torch.rand((40, nx), dtype=torch.float64, device="cuda")
    b3 = torch.zeros_like(a3)
    for ext in ((1, 1, 1, 1), (2, 1, 1, 2), (5, 5, 5, 5)):
        plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                              sg.FunctionStencil(sg.Extents(*ext), "san_fn", [0.5]), a3, b3, 1, 1)
        sg.compute(plan)
        sg.destroy_plan(plan)
# streamed host plan (ring of row chunks) and the opt-in partitioned CH sweeps
import os
os.environ["SG_STREAM_PLANS"], os.environ["SG_STREAM_ROWS"] = "1", "5"
gi = sg.Grid2D.from_array(rng.uniform(-1, 1, (23, 70)))
go = sg.Grid2D.from_array(np.zeros((23, 70)))
for mode in (sg.BoundaryMode.Periodic, sg.BoundaryMode.NonPeriodic):
    plan = sg.create_plan(sg.Direction.XY, mode, sg.WeightStencil(sg.Extents(2, 1, 1, 2), list(rng.uniform(-1, 1, 16))),
                          gi, go, 1, 1)
    sg.compute(plan)
    sg.destroy_plan(plan)
del os.environ["SG_STREAM_PLANS"], os.environ["SG_STREAM_ROWS"]
pp = sg.CHParams(nx=256, ny=256)
pp.dt = 0.1 * pp.dx()
pp.T = 1.0
sp = sg.CHStepper(pp)
sp.set_partition(4)
sp.step_many(3)
sp.synchronize()
# penta
for periodic in (True, False):
    m = sg.PentaBatch(70, 40, periodic)
    for band in m.bands():
        band[:] = rng.uniform(-1, 1, (40, 70))
    m.diag += 6.0
    f = sg.PeriodicPentaFactor(m) if periodic else sg.PentaFactor(m)
    t = torch.rand((40, 70), dtype=torch.float64, device="cuda")
    f.solve_in_place(t)
    u = sg.build_hyperdiffusion_operator(2.0, 64, 64, periodic)
    fu = sg.PeriodicPentaFactor(u) if periodic else sg.PentaFactor(u)
    tu = torch.rand((64, 64), dtype=torch.float64, device="cuda")
    fu.solve_in_place(tu)
# CH single GPU
p = sg.CHParams(nx=128, ny=128)
p.dt = 0.1 * p.dx()
p.T = 1.0
st = sg.CHStepper(p)
st.step_many(5)
st.step()
st.diagnostics()
# distributed CH, P2P, 2 simulated ranks
ranks = []
tr = LocalTransport(ranks)
for r in range(2):
    ranks.append(DistCHStepper(sg.CHParams(nx=256, ny=256, dt=0.1 * 2 * np.pi / 256, T=1.0), 2, r, transport=tr,
                               mode="p2p"))
for _ in range(2):
    for s_ in ranks:
        s_.phase_x()
    for s_ in ranks:
        s_.phase_y()
    for s_ in ranks:
        s_.phase_combine()
# slab stencil with fused P2P halos, 2 simulated ranks
kind = sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", list(rng.uniform(-1, 1, 9)))
sl = [SlabStencil(Slab(128, 64, 2, r, 1, 1, True), (1, 1, 1, 1), kind, torch.float64, "cuda") for r in range(2)]
tables = [[s_.p2p_buffers()[k] for s_ in sl] for k in range(2)]
for s_ in sl:
    s_.enable_p2p(tables, barrier=lambda: None)
for _ in range(2):
    for s_ in sl:
        s_.apply()
    for s_ in sl:
        s_.swap()
torch.cuda.synchronize()
print("workload OK")
