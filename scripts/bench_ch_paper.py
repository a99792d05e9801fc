"""The paper's own Cahn-Hilliard benchmark: step
to T = 10 on N x N, dt = 0.1 dx, D = 1, gamma = 0.01, uniform IC in +-0.1,
start-up and IO excluded — GPU (this library, full runs) against the
reference CHStepper on the host (oracle/_ref, serial and all cores; timed on
a bounded number of steps and scaled to T = 10, since the CPU is ~10^3x
slower). Prints one JSON line per N and a summary with the fitted time
exponents (the paper: CPU ~N^3, GPU N^2 -> N^3)."""
import json
import math
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    import paper_1902_09931_b200 as sg
    from oracle.oracle import Reference
    sizes = [int(x) for x in sys.argv[1:]] or [64, 128, 256, 512, 1024, 2048, 4096]
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    ref = Reference()
    rows = []
    for n in sizes:
        p = sg.CHParams(nx=n, ny=n)
        p.dt = 0.1 * p.dx()
        p.T = 10.0
        steps = int(math.ceil(p.T / p.dt - 1e-9))
        st = sg.CHStepper(p)
        st.step_many(3)
        st.synchronize()
        st.set_state(st.field(), st.previous_field())
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st.step_many(steps)
        st.synchronize()
        gpu = time.perf_counter() - t0
        rp = dict(D=p.D, gamma=p.gamma, lx=p.lx, ly=p.ly, dt=p.dt, T=p.T, nx=n, ny=n, seed=1, amp=0.1,
                  nonlinear=True)
        k = max(2, min(steps, int(2e8 // (n * n))))  # bounded CPU sample (~2e8 point-steps)
        serial = ref.ch_timed(rp, k, warmup=1, tiles=1, workers=1) * steps  # ch_timed: seconds per step
        k2 = max(2, min(steps, int(1e9 // (n * n))))
        par = ref.ch_timed(rp, k2, warmup=1, tiles=cores, workers=cores) * steps
        row = {"N": n, "steps_to_T10": steps, "gpu_s": gpu, "cpu_serial_s": serial, "cpu_parallel_s": par,
               "cores": cores, "speedup_vs_serial": serial / gpu, "speedup_vs_parallel": par / gpu,
               "cpu_sampled_steps": {"serial": k, "parallel": k2}}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del st
        torch.cuda.empty_cache()

    def slope(key):
        x = np.log([r["N"] for r in rows])
        y = np.log([r[key] for r in rows])
        return float(np.polyfit(x, y, 1)[0])

    print(json.dumps({"summary": "CH to T=10 (paper protocol)", "gpu_time_exponent": slope("gpu_s"),
                      "cpu_serial_time_exponent": slope("cpu_serial_s"),
                      "paper_claims": "GPU vs serial CPU O(10), ~40x at large N (Titan X Pascal vs i7-6850K)"}),
          flush=True)


if __name__ == "__main__":
    main()
