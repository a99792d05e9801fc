for rs in 128 256; do echo "RS $rs:"; SG_SWEEP_RS=$rs scripts/micro/sweep_trace 1024 | head -4; SG_SWEEP_RS=$rs timeout 120 python scripts/chtime.py 1024; done
SG_SWEEP_RS=256 timeout 900 python -m pytest tests/test_penta_gpu.py tests/test_ch_gpu.py -q -m gpu -x > gpurun_out/pytest_s2_11.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_s2_11.log
