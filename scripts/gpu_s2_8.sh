python scripts/exp/bigdebug2.py
timeout 900 python -m pytest tests/test_stencil_gpu.py tests/test_penta_gpu.py tests/test_ch_gpu.py -q -m gpu -x > gpurun_out/pytest_s2_8.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_s2_8.log
timeout 120 python scripts/chtime.py
