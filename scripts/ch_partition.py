"""Opt-in partitioned CH sweeps (sg_ch_set_partition): deviation from the
bitwise path (= the unmodified reference CHStepper, tests/test_ch_gpu.py)
after 100 steps, and steps/s, per grid and segment count. Also the x-sweep
of config 5's per-GPU share at G = 8 (1024 systems of 8192 unknowns): an
8192 x 1024 grid, whose x-sweep is exactly that batch.
Writes one JSON object per line (profiles/r02_ch_partition.jsonl)."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_1902_09931_b200 as sg


def stepper(nx, ny, P):
    p = sg.CHParams(nx=nx, ny=ny)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    st = sg.CHStepper(p)
    if P:
        st.set_partition(P)
    return st


def timed(st, k):
    st.step_many(5)
    st.synchronize()
    t = time.perf_counter()
    st.step_many(k)
    st.synchronize()
    return (time.perf_counter() - t) / k


out = []
for nx, ny, parts in ((1024, 1024, (2, 4, 8, 16)), (2048, 2048, (2, 4, 8)), (8192, 8192, (2, 4, 8, 16)),
                      (8192, 1024, (2, 4, 8, 16))):
    base = stepper(nx, ny, 0)
    base.step_many(100)
    c0 = base.field().values.copy()
    k = 1000 if nx * ny <= 2048 * 2048 else 50
    t0 = timed(stepper(nx, ny, 0), k)
    out.append({"nx": nx, "ny": ny, "P": 0, "us_per_step": t0 * 1e6, "steps_s": 1 / t0, "rel_l2_100": 0.0})
    for P in parts:
        st = stepper(nx, ny, P)
        st.step_many(100)
        c1 = st.field().values
        err = float(np.linalg.norm(c1 - c0) / np.linalg.norm(c0))
        t = timed(stepper(nx, ny, P), k)
        out.append({"nx": nx, "ny": ny, "P": P, "us_per_step": t * 1e6, "steps_s": 1 / t, "rel_l2_100": err})
    for o in out[-len(parts) - 1:]:
        print(json.dumps(o), flush=True)
