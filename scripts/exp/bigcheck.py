"""Debug: sampled-row parity of the 3x3 periodic fn stencil at growing sizes."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1902_09931_b200 as sg
from oracle.oracle import Restatement
orc = Restatement()
rng = np.random.default_rng(44)
w = list(rng.uniform(-1, 1, 9))
kind = sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", w)
for (ny, nx) in [(2048, 2048), (4096, 8192), (8192, 8192), (16384, 16384), (32768, 16384), (16384, 32768), (32768, 32768)]:
    g = torch.Generator(device="cuda").manual_seed(44)
    a = torch.rand((ny, nx), dtype=torch.float64, device="cuda", generator=g).mul_(2).sub_(1)
    b = torch.zeros_like(a)
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, kind, a, b, 1, 1)
    sg.compute(plan)
    torch.cuda.synchronize()
    bad = []
    for j in [0, 1, 511, 512, ny // 2, ny - 1]:
        band = np.stack([a[(j + d) % ny].cpu().numpy() for d in (-1, 0, 1)])
        want = orc.stencil(band, (1, 1, 1, 1), w, fn="fn_weighted_3x3")[1]
        got = b[j].cpu().numpy()
        if not np.array_equal(got.view(np.uint64), want.view(np.uint64)):
            bad.append((j, float(np.max(np.abs(got - want))), int(np.sum(got != want))))
    print(ny, nx, "kind", plan.kernel_kind(), "bad", bad, flush=True)
    sg.destroy_plan(plan)
    del a, b
    torch.cuda.empty_cache()
