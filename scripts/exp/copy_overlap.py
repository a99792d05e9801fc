"""PCIe copy overlap probe: H2D alone, D2H alone, both on two streams."""
import sys, time
sys.path.insert(0, ".")
import torch
n = 32768 * 32768
hin = torch.empty(n, dtype=torch.float64, pin_memory=True)
hout = torch.empty(n, dtype=torch.float64, pin_memory=True)
print("pinned", hin.is_pinned(), hout.is_pinned(), hin[5:100].is_pinned())
da = torch.empty(n, dtype=torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
C = 16
def chunks(x):
    return [x[n * c // C:n * (c + 1) // C] for c in range(C)]
def run(h2d, d2h):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if h2d:
        with torch.cuda.stream(s1):
            for d, h in zip(chunks(da), chunks(hin)):
                d.copy_(h, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2):
            for h, d in zip(chunks(hout), chunks(db)):
                h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0
for rep in range(2):
    a, b, c = run(1, 0), run(0, 1), run(1, 1)
    gb = n * 8 / 1e9
    print(f"H2D {gb/a:.1f} GB/s  D2H {gb/b:.1f} GB/s  both {2*gb/c:.1f} GB/s aggregate ({c*1e3:.0f} ms)", flush=True)
