mkdir -p gpurun_out
echo "PDL on:"; timeout 120 python scripts/chtime.py
echo "PDL off:"; SG_PDL=0 timeout 120 python scripts/chtime.py
echo "PDL on:"; timeout 120 python scripts/chtime.py 1024
timeout 600 python -m pytest tests/test_ch_gpu.py tests/test_penta_gpu.py tests/test_diagnostics_gpu.py -x -q -m gpu > gpurun_out/pytest_s2_3.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_s2_3.log
