timeout 900 python -m pytest tests/test_diagnostics_gpu.py tests/test_weno_gpu.py tests/test_stencil_gpu.py -q -m gpu -x > gpurun_out/pytest_ab3.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_ab3.log
python -c "
import sys, time; sys.path.insert(0,'.')
import paper_1902_09931_b200 as sg
p = sg.CHParams(nx=1024, ny=1024); p.dt = 0.1*p.dx(); p.T = 1.0
st = sg.CHStepper(p); st.step_many(10); st.diagnostics()
t=time.perf_counter()
for _ in range(20): d = st.diagnostics()
print('diagnostics 1024^2: %.3f ms/call' % ((time.perf_counter()-t)/20*1e3))
"
