"""Does recording per-launch events change the measured stencil time?"""
import statistics, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1902_09931_b200 as sg
from bench import time_plan_steps
NX = NY = 32768
a = torch.rand((NY, NX), dtype=torch.float64, device="cuda").mul_(2).sub_(1)
b = torch.empty_like(a)
w = list(np.random.default_rng(4).uniform(-1, 1, 9))
plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", w), a, b, 1, 1)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for rep in range(3):
        tot, per = time_plan_steps(sg, torch, plan, 100, s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(100):
            sg.compute(plan, stream=s, synchronize=False); sg.swap_plan(plan)
        e1.record(s); e1.synchronize()
        t2 = e0.elapsed_time(e1)
        print(f"with events: {tot/100:.4f} ms/step (mean launch {statistics.mean(per):.4f});  without: {t2/100:.4f} ms/step", flush=True)
