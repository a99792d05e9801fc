"""How far the CH field moves under a mere change of rounding order: run
`steps` steps at n^2 with whatever library SG_LIB_PATH selects and save C^n
(python ch_fma_sensitivity.py n steps out.npy). Run once with the faithful
build and once with the same kernels built with --fmad=true (FMA
contraction): their relative L2 distance is the scale against which any
reordered algorithm (the partitioned sweeps) is measured — the SURVEY's
probe of the CPU reference found the same effect (2.3e-11 after 100 steps
at 1024^2)."""
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_1902_09931_b200 as sg

n, steps, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
p = sg.CHParams(nx=n, ny=n)
p.dt = 0.1 * p.dx()
p.T = 1.0
st = sg.CHStepper(p)
st.step_many(steps)
np.save(out, st.field().values)
