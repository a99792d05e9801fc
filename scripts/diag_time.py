"""CH diagnostics() cost against the step time (1024^2, 4096^2, 8192^2)."""
import sys, time
sys.path.insert(0, ".")
import paper_1902_09931_b200 as sg
for n in (1024, 4096, 8192):
    p = sg.CHParams(nx=n, ny=n); p.dt = 0.1 * p.dx(); p.T = 1.0
    st = sg.CHStepper(p); st.step_many(3); st.synchronize()
    st.diagnostics()
    t = time.perf_counter()
    for _ in range(10): d = st.diagnostics()
    dt = (time.perf_counter() - t) / 10
    t = time.perf_counter(); st.step_many(20); st.synchronize(); ds = (time.perf_counter() - t) / 20
    print(f"n={n}: diagnostics {dt*1e3:.3f} ms (= {dt/ds:.1f} steps), step {ds*1e6:.1f} us", flush=True)
    del st
