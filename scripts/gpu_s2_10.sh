scripts/micro/sweep_trace 1024 | head -5
echo "RS auto:"; timeout 120 python scripts/chtime.py
echo "RS 64:"; SG_SWEEP_RS=64 timeout 120 python scripts/chtime.py 1024
timeout 900 python -m pytest tests/test_penta_gpu.py tests/test_ch_gpu.py -q -m gpu -x > gpurun_out/pytest_s2_10.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_s2_10.log
