"""FP32 / FP64 A/B of a few shapes on odd and even 16384-wide grids (SG_LIB_PATH)."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch

import paper_1902_09931_b200 as sg

n = 16384
rng = np.random.default_rng(0)
for dt, esz in ((torch.float32, 4), (torch.float64, 8)):
    a = torch.rand((n, n), dtype=dt, device="cuda")
    b = torch.zeros_like(a)
    for nxv in (n, n - 1):
        ai = a.view(-1)[: n * nxv].view(n, nxv)
        bo = b.view(-1)[: n * nxv].view(n, nxv)
        for ext, fn in (((1, 1, 1, 1), "fn_weighted_3x3"), ((2, 1, 1, 2), None), ((3, 1, 0, 0), None), ((2, 2, 2, 2), None)):
            nv = 9 if fn else (ext[0] + ext[1] + 1) * (ext[2] + ext[3] + 1)
            e = sg.Extents(*ext)
            kind = sg.FunctionStencil(e, fn, list(rng.uniform(-1, 1, 9))) if fn else sg.WeightStencil(e, list(rng.uniform(-1, 1, nv)))
            plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, kind, ai, bo, 1, 1)
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
            print(json.dumps({"dt": esz, "ext": ext, "nx": nxv, "kind": plan.kernel_kind(),
                              "hbm": round(2 * esz * n * nxv / (ms * 1e-3) / 1e9 / 6544, 3)}), flush=True)
            sg.destroy_plan(plan)
    del a, b
    torch.cuda.empty_cache()
