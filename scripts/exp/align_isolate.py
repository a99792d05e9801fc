"""Isolate k_tma_g's misalignment costs at 16384^2: input / output pointer
phase (constant per row) vs row-varying phase (odd nx), per dtype.
usage: python scripts/exp/align_isolate.py float32|float64 [ext...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1902_09931_b200 as sg

dt = getattr(torch, sys.argv[1] if len(sys.argv) > 1 else "float32")
n = 16384
rng = np.random.default_rng(0)
A = torch.rand(n * n + 64, dtype=dt, device="cuda")
B = torch.zeros_like(A)
cases = [("aligned", n, 0, 0), ("in+1", n, 1, 0), ("out+1", n, 0, 1), ("both+1", n, 1, 1),
         ("in+2", n, 2, 0), ("out+2", n, 0, 2), ("odd_nx", n - 1, 0, 0), ("nx-2", n - 2, 0, 0)]
for ext in ((0, 0, 0, 0), (1, 1, 1, 1)):
    for name, nx, oi, oo in cases:
        ai = A[oi:oi + n * nx].view(n, nx)
        bo = B[oo:oo + n * nx].view(n, nx)
        nv = (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
        plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                              sg.WeightStencil(sg.Extents(*ext), list(rng.uniform(-1, 1, nv))), ai, bo, 1, 1)
        for _ in range(3):
            sg.compute(plan, synchronize=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(30):
            sg.compute(plan, synchronize=False)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 30
        print(sys.argv[1] if len(sys.argv) > 1 else "float32", ext, name, plan.kernel_kind(),
              round(2 * A.element_size() * n * nx / (ms * 1e-3) / 1e9 / 6544, 3), flush=True)
        sg.destroy_plan(plan)
