timeout 600 python -m pytest tests/test_p2p_ipc_gpu.py -q -m gpu -x > gpurun_out/pytest_ab13.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_ab13.log
