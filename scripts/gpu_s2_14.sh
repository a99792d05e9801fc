echo "xin:"; timeout 120 python scripts/chtime.py
echo "no xin:"; SG_CH_XIN=0 timeout 120 python scripts/chtime.py
timeout 900 python -m pytest tests/test_ch_gpu.py tests/test_penta_gpu.py tests/test_diagnostics_gpu.py -q -m gpu -x > gpurun_out/pytest_s2_14.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_s2_14.log
