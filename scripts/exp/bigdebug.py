"""Debug: identity 3x3 weight stencil on a[j][i] = j; which rows come back wrong?"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1902_09931_b200 as sg
idw = [0, 0, 0, 0, 1.0, 0, 0, 0, 0]
for (ny, nx) in [(32768, 1024), (32768, 2048), (24576, 1024), (16384 + 512, 1024), (65536, 1024)]:
    a = torch.arange(ny, dtype=torch.float64, device="cuda")[:, None].repeat(1, nx).contiguous()
    b = torch.full_like(a, -1.0)
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                          sg.WeightStencil(sg.Extents(1, 1, 1, 1), idw), a, b, 1, 1)
    sg.compute(plan)
    torch.cuda.synchronize()
    bad = (b != a).any(dim=1).nonzero().flatten().cpu().numpy()
    msg = f"{ny}x{nx}: {len(bad)} bad rows"
    if len(bad):
        j = bad[:8]
        msg += f" first {j.tolist()} got {b[j, 0].cpu().numpy().tolist()} last {bad[-3:].tolist()}"
    print(msg, flush=True)
    sg.destroy_plan(plan)
