"""One stencil plan at 16384^2 for ncu captures: dtype ext(l,r,t,b) in_off out_off nx [reps]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1902_09931_b200 as sg

dt = getattr(torch, sys.argv[1])
ext = tuple(int(x) for x in sys.argv[2].split(","))
oi, oo, nx = int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
n = 16384
A = torch.rand(n * n + 64, dtype=dt, device="cuda")
B = torch.zeros_like(A)
nv = (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                      sg.WeightStencil(sg.Extents(*ext), list(np.random.default_rng(0).uniform(-1, 1, nv))),
                      A[oi:oi + n * nx].view(n, nx), B[oo:oo + n * nx].view(n, nx), 1, 1)
for _ in range(reps):
    sg.compute(plan, synchronize=False)
torch.cuda.synchronize()
print("kind", plan.kernel_kind())
