"""CH steps/s (single GPU stepper). Usage: chtime.py [n ...]; SG_PART=P
times the opt-in partitioned sweeps with P segments per system as well."""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_1902_09931_b200 as sg

sizes = [int(x) for x in sys.argv[1:]] or [1024, 8192]
parts = [0] + [int(v) for v in os.environ.get("SG_PART", "").split(",") if v]
for n in sizes:
    for P in parts:
        p = sg.CHParams(nx=n, ny=n)
        p.dt = 0.1 * p.dx()
        p.T = 1.0
        st = sg.CHStepper(p)
        if P:
            try:
                st.set_partition(P)
            except Exception as e:  # noqa: BLE001
                print(f"CH {n}^2 P={P}: unavailable ({e})")
                continue
        st.step_many(10)
        st.synchronize()
        k = 1000 if n <= 2048 else 40
        t = time.perf_counter()
        st.step_many(k)
        st.synchronize()
        dt = time.perf_counter() - t
        print(f"CH {n}^2 P={P}: {k / dt:.1f} steps/s ({dt / k * 1e6:.1f} us/step)", flush=True)
