"""Headline config (32768^2 XY periodic fn_weighted_3x3) FP64 and FP32,
kernel time per launch over 100 launches — for A/B of builds
(SG_LIB_PATH). Prints one JSON line per dtype."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch

import paper_1902_09931_b200 as sg

n = 32768
w = list(np.random.default_rng(0).uniform(-1, 1, 9))
for dt in (torch.float64, torch.float32):
    a = torch.rand((n, n), dtype=dt, device="cuda")
    b = torch.empty_like(a)
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                          sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", w), a, b, 1, 1)
    for _ in range(5):
        sg.compute(plan, synchronize=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        sg.compute(plan, synchronize=False)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 100
    print(json.dumps({"lib": os.path.basename(os.environ.get("SG_LIB_PATH", "default")), "dtype": str(dt),
                      "ms": round(ms, 4), "gpts": round(n * n / ms / 1e6, 1)}), flush=True)
    sg.destroy_plan(plan)
    del a, b
    torch.cuda.empty_cache()
