"""Debug: random 3x3 periodic stencil vs a torch roll reference, full grid."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1902_09931_b200 as sg
rng = np.random.default_rng(44)
w = list(rng.uniform(-1, 1, 9))

def ref(a):
    out = torch.zeros_like(a)
    for q in range(3):
        for p in range(3):
            out += w[q * 3 + p] * torch.roll(a, shifts=(1 - q, 1 - p), dims=(0, 1))
    return out

for (ny, nx, how) in [(32768, 2048, "randgen"), (32768, 2048, "rand"), (32768, 16384, "rand"), (32768, 16384, "randgen"),
                      (16384, 16384, "randgen")]:
    if how == "randgen":
        g = torch.Generator(device="cuda").manual_seed(44)
        a = torch.rand((ny, nx), dtype=torch.float64, device="cuda", generator=g).mul_(2).sub_(1)
    else:
        a = torch.rand((ny, nx), dtype=torch.float64, device="cuda").mul_(2).sub_(1)
    for kname in ["fn", "w"]:
        b = torch.zeros_like(a)
        kind = (sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", w) if kname == "fn"
                else sg.WeightStencil(sg.Extents(1, 1, 1, 1), w))
        plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, kind, a, b, 1, 1)
        sg.compute(plan)
        torch.cuda.synchronize()
        r = ref(a)
        err = (b - r).abs().amax(dim=1)
        bad = (err > 1e-12).nonzero().flatten().cpu().numpy()
        msg = f"{ny}x{nx} {how} {kname}: {len(bad)} bad rows"
        if len(bad):
            msg += f" first {bad[:6].tolist()} last {bad[-3:].tolist()}"
            # which input row-shift explains row bad[0]?
            j = int(bad[0])
            for s in range(-3, 4):
                rr = ref(torch.roll(a, shifts=s, dims=0))
                if (b[j] - rr[j]).abs().max() < 1e-12:
                    msg += f" (row {j} matches shift {s})"
        print(msg, flush=True)
        sg.destroy_plan(plan)
        del b
    del a
    torch.cuda.empty_cache()
