"""CH steps/s at 1024^2 and 8192^2 (single GPU stepper)."""
import sys, time
sys.path.insert(0, ".")
import paper_1902_09931_b200 as sg
sizes = [int(x) for x in sys.argv[1:]] or [1024, 8192]
for n in sizes:
    p = sg.CHParams(nx=n, ny=n); p.dt = 0.1 * p.dx(); p.T = 1.0
    st = sg.CHStepper(p); st.step_many(10); st.synchronize()
    k = 1000 if n <= 2048 else 40
    t = time.perf_counter(); st.step_many(k); st.synchronize(); dt = time.perf_counter() - t
    print(f"CH {n}^2: {k/dt:.1f} steps/s ({dt/k*1e6:.1f} us/step)", flush=True)
