"""Timeline of the merged CH RHS + x-sweep kernel (build with -DSG_MERGE_TRACE,
SG_LIB_PATH=build/libT.so): per tile publish time, per sweep CTA stage-ready
times, relative to the earliest CTA start."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np

import paper_1902_09931_b200 as sg
from paper_1902_09931_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
p = sg.CHParams(nx=n, ny=n)
p.dt = 0.1 * p.dx()
p.T = 1.0
st = sg.CHStepper(p)
st.step_many(3)  # head, one merged steady step, tail
st.synchronize()
buf = (C.c_ulonglong * 8192)()
_lib.lib().sg_debug_merge_trace.argtypes = [C.c_void_p, C.c_int]
_lib.lib().sg_debug_merge_trace(buf, 8192)
a = np.array(buf, dtype=np.float64)
tilesX, tilesY = n // 64, n // 32
nsweep = n // 32
cta_start = a[4096:4096 + 2 * 148:2]
cta_start = cta_start[cta_start > 0]
t0 = cta_start.min()
tiles = (a[:tilesX * tilesY] - t0) / 1e3
ends = a[4097:4096 + 2 * 148:2]
sw_end = (ends[:nsweep] - t0) / 1e3
rhs_end = (ends[nsweep:][ends[nsweep:] > 0] - t0) / 1e3
print("sweep CTA end (us): min %.2f max %.2f; RHS CTA end: min %.2f max %.2f" % (sw_end.min(), sw_end.max(),
      rhs_end.min(), rhs_end.max()))
print("CTA start spread (us): %.2f .. %.2f" % (0, (cta_start.max() - t0) / 1e3))
print("tile publish (us): min %.2f median %.2f max %.2f" % (tiles.min(), np.median(tiles), tiles.max()))
tl = tiles.reshape(tilesY, tilesX)
print("per tile column, latest publish (us):", " ".join("%.1f" % v for v in tl.max(axis=0)))
sw = a[4096 + 512:4096 + 512 + nsweep * 64].reshape(nsweep, 64)
stages = n // 128
sw = (sw[:, :stages] - t0) / 1e3
print("sweep stage-ready (us), CTA 0:", " ".join("%.1f" % v for v in sw[0]))
print("sweep stage-ready (us), max over CTAs:", " ".join("%.1f" % v for v in sw.max(axis=0)))
