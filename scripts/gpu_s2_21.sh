timeout 120 python scripts/chtime.py
timeout 900 python -m pytest tests/test_ch_gpu.py tests/test_penta_gpu.py tests/test_ch_dist_gpu.py -q -m gpu -x > gpurun_out/pytest_s2_21.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_s2_21.log
