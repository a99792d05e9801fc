mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ch_gpu.py tests/test_penta_gpu.py tests/test_ch_dist_gpu.py -x -q -m gpu > gpurun_out/pytest_gpu18.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu18.log
cat > /tmp/chtime.py <<'PY'
import time, sys
sys.path.insert(0, '.')
import paper_1902_09931_b200 as sg
for n in (1024, 8192):
    p = sg.CHParams(nx=n, ny=n); p.dt = 0.1 * p.dx(); p.T = 1.0
    st = sg.CHStepper(p); st.step_many(10); st.synchronize()
    k = 1000 if n <= 2048 else 40
    t = time.perf_counter(); st.step_many(k); st.synchronize(); dt = time.perf_counter() - t
    print(f"CH {n}^2: {k/dt:.1f} steps/s ({dt/k*1e6:.1f} us/step)")
PY
python /tmp/chtime.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ch1024_launches18.csv python scripts/profile_ch.py --n 1024 --steps 5 > /dev/null 2>&1; echo ncu=$?
