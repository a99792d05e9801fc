import json, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1902_09931_b200 as sg
n = 16384
rng = np.random.default_rng(0)
a = torch.rand((n, n), dtype=getattr(torch, sys.argv[1] if len(sys.argv) > 1 else "float32"), device="cuda"); b = torch.zeros_like(a)
for nxv in (n, n - 1, n - 2):
    ai = a.view(-1)[: n * nxv].view(n, nxv); bo = b.view(-1)[: n * nxv].view(n, nxv)
    for ext in ((0, 0, 0, 0), (1, 1, 0, 0), (0, 0, 1, 1), (1, 1, 1, 1)):
        nv = (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
        plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, sg.WeightStencil(sg.Extents(*ext), list(rng.uniform(-1, 1, nv))), ai, bo, 1, 1)
        for _ in range(3): sg.compute(plan, synchronize=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(30): sg.compute(plan, synchronize=False)
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 30
        print(nxv, ext, plan.kernel_kind(), round(2 * a.element_size() * n * nxv / (ms * 1e-3) / 1e9 / 6544, 3), flush=True)
        sg.destroy_plan(plan)
