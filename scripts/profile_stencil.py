"""Run a few applications of one stencil config (for ncu captures).

python scripts/profile_stencil.py [--dtype f64|f32] [--n 32768] [--fn fn_weighted_3x3|weights]
                                  [--ext 1,1,1,1] [--reps 5]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_1902_09931_b200 as sg

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="f64")
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--ny", type=int, default=0)
ap.add_argument("--fn", default="fn_weighted_3x3")
ap.add_argument("--ext", default="1,1,1,1")
ap.add_argument("--periodic", type=int, default=1)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
sg._lib.check(sg._lib.lib().sg_init(0))
ny = a.ny or a.n
dt = torch.float64 if a.dtype == "f64" else torch.float32
x = torch.rand((ny, a.n), dtype=dt, device="cuda")
y = torch.zeros_like(x)
ext = sg.Extents(*[int(v) for v in a.ext.split(",")])
W = ext.width() * ext.height()
w = list(np.random.default_rng(0).uniform(-1, 1, W if a.fn == "weights" else 9))
kind = sg.WeightStencil(ext, w) if a.fn == "weights" else sg.FunctionStencil(ext, a.fn, w)
d = 0 if ext.top == 0 and ext.bottom == 0 else (1 if ext.left == 0 and ext.right == 0 else 2)
plan = sg.create_plan(d, 0 if a.periodic else 1, kind, x, y, 1, 1)
print("kernel kind", plan.kernel_kind())
for _ in range(a.reps):
    sg.compute(plan)
torch.cuda.synchronize()
print("done")
