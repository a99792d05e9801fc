import sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1902_09931_b200 as sg
periodic = sys.argv[1] == "1"; B = int(sys.argv[2]); n = int(sys.argv[3])
m = sg.build_hyperdiffusion_operator(2.5, n, B, periodic)
rhs = np.random.default_rng(n).uniform(-1, 1, (n, B))
f = sg.PeriodicPentaFactor(m) if periodic else sg.PentaFactor(m)
t = torch.from_numpy(rhs.copy()).cuda()
f.solve_in_place(t)
torch.cuda.synchronize()
print("ok", periodic, B, n)
