timeout 900 python -m pytest tests/test_slab_gpu.py -q -m gpu -x > gpurun_out/pytest_ab7.log 2>&1; echo pytest=$?; tail -25 gpurun_out/pytest_ab7.log
