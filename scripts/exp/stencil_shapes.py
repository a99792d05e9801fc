"""Time stencil shapes on a 16384^2 FP64 grid (device tensors) — A/B of
build variants selected by SG_LIB_PATH. Prints one JSON line per shape."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch

import paper_1902_09931_b200 as sg

n = 16384
peak = json.loads((Path(__file__).resolve().parents[2] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (Path(__file__).resolve().parents[2] / "MEASURED_PEAKS.json").exists() else 6544.0
shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]] or [
    (3, 1, 0, 0), (2, 1, 1, 2), (2, 2, 2, 2), (4, 4, 4, 4), (1, 1, 1, 1), (2, 2, 0, 0), (1, 2, 2, 1), (2, 2, 2, 1),
    (3, 3, 3, 3), (0, 0, 2, 2)]
DT = torch.float32 if os.environ.get("SG_DT") == "f32" else torch.float64
ESZ = 4 if DT == torch.float32 else 8
a = torch.rand((n, n), dtype=DT, device="cuda")
b = torch.zeros_like(a)
rng = np.random.default_rng(0)
for odd in (False, True):
    nxv = n - 1 if odd else n
    ai = a.view(-1)[: n * nxv].view(n, nxv)
    bo = b.view(-1)[: n * nxv].view(n, nxv)
    for ext in shapes:
        l, r, t, bb = ext
        nv = (l + r + 1) * (t + bb + 1)
        plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                              sg.WeightStencil(sg.Extents(*ext), list(rng.uniform(-1, 1, nv))), ai, bo, 1, 1)
        for _ in range(3):
            sg.compute(plan, synchronize=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 30
        e0.record()
        for _ in range(reps):
            sg.compute(plan, synchronize=False)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"lib": os.environ.get("SG_LIB_PATH", "default"), "ext": ext, "nx": nxv,
                          "kind": plan.kernel_kind(), "ms": round(ms, 4),
                          "hbm_frac": round(2 * ESZ * n * nxv / (ms * 1e-3) / 1e9 / peak, 4), "esz": ESZ,
                          "fp64_ops": 2 * nv}), flush=True)
        sg.destroy_plan(plan)
