timeout 120 python scripts/chtime.py; timeout 120 python scripts/chtime.py 1024 256 128
timeout 600 python -m pytest tests/test_ch_gpu.py -q -m gpu -x -k "steady or 1000 or tolerance" > gpurun_out/pytest_ab14.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_ab14.log
