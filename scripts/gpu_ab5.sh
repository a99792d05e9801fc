timeout 1200 python -m pytest tests/test_ch_gpu.py -q -m gpu -x -k "reference" --durations=3 > gpurun_out/pytest_ab5.log 2>&1; echo pytest=$?; tail -8 gpurun_out/pytest_ab5.log
