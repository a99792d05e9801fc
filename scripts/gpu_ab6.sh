timeout 1200 python -m pytest tests/test_stencil_gpu.py -q -m gpu -x -k "full" --durations=5 > gpurun_out/pytest_ab6.log 2>&1; echo pytest=$?; tail -12 gpurun_out/pytest_ab6.log
