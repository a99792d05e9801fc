"""General (per-system) periodic penta solve on the device vs the reference."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1902_09931_b200 as sg
from oracle.oracle import Reference
B, n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192, 1024
rng = np.random.default_rng(1)
for periodic in (True, False):
    m = sg.PentaBatch(B, n, periodic)
    for band in m.bands():
        band[:] = rng.uniform(-1, 1, (n, B))
    m.diag += 6.0
    t0 = time.perf_counter()
    f = sg.PeriodicPentaFactor(m) if periodic else sg.PentaFactor(m)
    torch.cuda.synchronize()
    tf = time.perf_counter() - t0
    rhs = torch.rand((n, B), dtype=torch.float64, device="cuda")
    for _ in range(3):
        f.solve_in_place(rhs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f.solve_in_place(rhs)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    # bytes: factor tables (m1 m2 dInv ap bp [+W0..3]) read once, z read+written twice
    tables = 5 + (4 if periodic else 0)
    gb = (tables * B * n * 8 + 4 * B * n * 8) / 1e9
    ref = Reference()
    cores = len(os.sched_getaffinity(0))
    rb = rng.uniform(-1, 1, (n, B))
    t0 = time.perf_counter()
    ref.penta_solve(periodic, m.bands(), rb, workers=cores)
    tr = time.perf_counter() - t0
    print(f"periodic={periodic} B={B} n={n}: device factor {tf*1e3:.1f} ms (incl. H2D), solve {ms:.3f} ms "
          f"({gb/ms*1e3:.0f} GB/s), reference factor+solve {tr*1e3:.0f} ms on {cores} cores", flush=True)
