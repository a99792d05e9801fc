scripts/micro/sweep_trace 1024 | head -8; scripts/micro/sweep_trace 8192 | head -8
timeout 600 python -m pytest tests/test_penta_gpu.py tests/test_ch_gpu.py tests/test_ch_dist_gpu.py -x -q -m gpu --timeout 120 > gpurun_out/pytest_gpu28.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu28.log
timeout 120 python scripts/chtime.py
