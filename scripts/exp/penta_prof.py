import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1902_09931_b200 as sg
B, n = int(sys.argv[1]), 1024
periodic = sys.argv[2] == "1"
rng = np.random.default_rng(1)
m = sg.PentaBatch(B, n, periodic)
for band in m.bands():
    band[:] = rng.uniform(-1, 1, (n, B))
m.diag += 6.0
f = sg.PeriodicPentaFactor(m) if periodic else sg.PentaFactor(m)
rhs = torch.rand((n, B), dtype=torch.float64, device="cuda")
for _ in range(3):
    f.solve_in_place(rhs)
torch.cuda.synchronize()
