timeout 600 python -m pytest tests/test_ch_dist_gpu.py -q -m gpu -x > gpurun_out/pytest_s2_24.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_s2_24.log
